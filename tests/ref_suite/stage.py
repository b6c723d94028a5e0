"""Stage the reference's own test suite for the drop-in check (test infrastructure).

Copies ``/root/reference/pkg/tests`` and the reference package
``/root/reference/pkg/src/lodstream`` (its callers of the hot path: io, synth,
service, cli, ws) into ``tests/ref_suite/_ref/`` -- git-ignored, like
``oracle/_ref``: nothing of the reference enters the repository's history, but
the staged copy travels to the GPU box with the working tree (``/root/reference``
does not exist there).  ``__graft_entry__.build()`` runs this when the
reference is present.  The hot-path modules of the staged package (update,
render, octree, store) are never used: ``alias_plugin.py`` maps them onto the
B200 facade before anything imports them.
"""
from __future__ import annotations

import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
REFERENCE = os.environ.get("LOD_REFERENCE_ROOT", "/root/reference")


def stage(reference: str = REFERENCE) -> str | None:
    src_tests = os.path.join(reference, "pkg", "tests")
    src_pkg = os.path.join(reference, "pkg", "src", "lodstream")
    if not (os.path.isdir(src_tests) and os.path.isdir(src_pkg)):
        return None
    if os.path.isdir(DEST):
        shutil.rmtree(DEST)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc", "*.nbi", "*.nbc")
    shutil.copytree(src_tests, os.path.join(DEST, "tests"), ignore=ignore)
    shutil.copytree(src_pkg, os.path.join(DEST, "lodstream"), ignore=ignore)
    with open(os.path.join(DEST, "pytest.ini"), "w") as f:
        f.write("[pytest]\n")
    return DEST


if __name__ == "__main__":
    print(stage() or "reference not found")
