"""The C-ABI structure layouts, as the compiler lays them out from
include/lod_b200.h, against both ctypes bindings: the facade's
(paper_2310_03567_b200/_lib.py) and the reference-side binding a lodstream
maintainer would add (integration/lodstream_b200.py).  A
binding whose struct is shorter than the header's overruns the caller's
buffer on every call, so every field offset and every size is compared."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _c_layout(tmp_path, structs) -> dict:
    """{struct: {"__size__": n, field: offset}} from the C compiler."""
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lod_b200.h"', "int main(void) {"]
    for name, fields in structs.items():
        lines.append(f'  printf("{name} __size__ %zu\\n", sizeof({name}));')
        for f in fields:
            lines.append(f'  printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = line.split()
        out.setdefault(s, {})[f] = int(v)
    return out


def _bindings():
    import sys

    sys.path.insert(0, ROOT)
    from integration import lodstream_b200 as ref_side
    from paper_2310_03567_b200 import _lib

    return {
        "facade": {c.__name__: c for c in (_lib.LodParams, _lib.LodLimits, _lib.LodBatchStats, _lib.LodTreeInfo,
                                           _lib.LodDeltaInfo, _lib.LodSettleStats)},
        "integration": {c.__name__: c for c in ref_side.STRUCTS},
    }


@pytest.mark.parametrize("which", ["facade", "integration"])
def test_struct_layouts_match_header(tmp_path, which):
    structs = _bindings()[which]
    assert set(structs) == {"LodParams", "LodLimits", "LodBatchStats", "LodTreeInfo", "LodDeltaInfo",
                            "LodSettleStats"}
    c = _c_layout(tmp_path, {name: [f for f, _ in cls._fields_] for name, cls in structs.items()})
    for name, cls in structs.items():
        assert ctypes.sizeof(cls) == c[name]["__size__"], (which, name, ctypes.sizeof(cls), c[name]["__size__"])
        for f, _ in cls._fields_:
            assert getattr(cls, f).offset == c[name][f], (which, name, f)


def test_integration_binding_loads_and_types_every_symbol():
    import sys

    sys.path.insert(0, ROOT)
    from integration import lodstream_b200 as ref_side

    so = os.path.join(ROOT, "paper_2310_03567_b200", "_lodb200.so")
    if not os.path.exists(so):
        pytest.skip("library not built")
    L = ref_side.lib(so)
    for name in ref_side._SIGS:
        assert getattr(L, name).argtypes is not None, name
    assert L.lod_strerror(1) == b"arena exhausted"
    assert ref_side.ERRORS == {1: "OutOfArena", 2: "SpillOverflow", 3: "BacklogOverflow"}
