"""pytest plugin: run the reference's own tests against the B200 path.

Loaded with ``-p alias_plugin`` before any test module is imported.  It puts
the staged reference package (``_ref/lodstream``: io, synth, service, cli, ws
-- the callers of the hot path) on ``sys.path`` and pre-registers the hot-path
modules under the reference's names, so every ``from lodstream.update import
insert_batch`` / ``lodstream.render`` / ``lodstream.octree`` /
``lodstream.store`` in the tests and in the reference's own callers (service
binds ``insert_batch`` at import, service.py:42) resolves to the B200 facade
(``paper_2310_03567_b200``).  ``lodstream.errors`` stays the reference module
(io's format errors live there) with its three fatal exceptions replaced by
the facade's, which ``insert_batch`` raises.
"""
from __future__ import annotations

import importlib.util
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")
ROOT = os.path.dirname(os.path.dirname(HERE))


def _composite(name: str, mod):
    """Module ``lodstream.<name>``: the reference module's namespace with every
    name the facade module defines replaced by the facade's."""
    import types

    full = "lodstream." + name
    spec = importlib.util.spec_from_file_location(f"lodstream._reference_{name}",
                                                  os.path.join(REF, "lodstream", name + ".py"))
    ref = importlib.util.module_from_spec(spec)
    ref.__package__ = "lodstream"
    sys.modules[spec.name] = ref
    spec.loader.exec_module(ref)
    comp = types.ModuleType(full, mod.__doc__)
    comp.__dict__.update({k: v for k, v in vars(ref).items() if not k.startswith("__")})
    comp.__dict__.update({k: v for k, v in vars(mod).items() if not k.startswith("__")})
    comp.__file__ = mod.__file__
    comp.__package__ = "lodstream"
    comp.__b200__ = mod
    return comp


def _install() -> None:
    if "lodstream" in sys.modules:
        return
    for p in (ROOT, REF, os.path.join(REF, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref_suite")
    from paper_2310_03567_b200 import errors as b_errors
    from paper_2310_03567_b200 import octree as b_octree
    from paper_2310_03567_b200 import render as b_render
    from paper_2310_03567_b200 import store as b_store
    from paper_2310_03567_b200 import update as b_update

    # the package object first, without running its __init__ (which imports
    # update / octree / store): the aliases must be in place before that
    import types

    pkg = types.ModuleType("lodstream")
    pkg.__path__ = [os.path.join(REF, "lodstream")]
    pkg.__file__ = os.path.join(REF, "lodstream", "__init__.py")
    pkg.__package__ = "lodstream"
    sys.modules["lodstream"] = pkg
    spec = importlib.util.spec_from_file_location("lodstream.errors", os.path.join(REF, "lodstream", "errors.py"))
    ref_errors = importlib.util.module_from_spec(spec)
    sys.modules["lodstream.errors"] = ref_errors
    spec.loader.exec_module(ref_errors)
    for name in ("OutOfArena", "SpillOverflow", "BacklogOverflow"):
        setattr(ref_errors, name, getattr(b_errors, name))
    # each hot-path module: the facade's names, over the reference module's
    # out-of-scope leftovers (e.g. render.write_image / overlay_node_boxes,
    # image output) so the tests import every name they expect
    for name, mod in (("store", b_store), ("octree", b_octree), ("update", b_update), ("render", b_render)):
        sys.modules["lodstream." + name] = _composite(name, mod)
    with open(pkg.__file__) as f:  # the package's own __init__, now binding the aliased modules
        exec(compile(f.read(), pkg.__file__, "exec"), pkg.__dict__)
    import lodstream

    assert lodstream.insert_batch is b_update.insert_batch and lodstream.Octree is b_octree.Octree
    for name in ("errors", "store", "octree", "update", "render"):
        setattr(lodstream, name, sys.modules["lodstream." + name])


_install()
