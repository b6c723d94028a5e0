"""CPU checks of the C-ABI boundary: the library builds, loads, exports every
symbol include/lod_b200.h declares, and the product fails loudly without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lod_b200.h")


def declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lod_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    from paper_2310_03567_b200 import _lib, build

    path = build.build()
    assert os.path.exists(path)
    L = _lib.load()
    assert isinstance(L, ctypes.CDLL)


def test_every_declared_symbol_is_exported_and_bound():
    from paper_2310_03567_b200 import _lib

    names = declared_functions()
    assert len(names) >= 20
    L = _lib.load()
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lod_[a-z0-9_]+)$", out, flags=re.M))
    assert set(names) <= exported, set(names) - exported


def test_library_targets_sm100a_only():
    from paper_2310_03567_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_struct_layouts_match_header():
    from paper_2310_03567_b200 import _lib

    assert ctypes.sizeof(_lib.LodParams) == 3 * 8 + 8 + 4 * 8 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.LodLimits) == 24
    assert ctypes.sizeof(_lib.LodBatchStats) == 15 * 8 + 4 + 4 + 4 * _lib.LOD_NPHASE
    assert ctypes.sizeof(_lib.LodTreeInfo) == 12 * 8


def test_no_cpu_fallback_without_device():
    import numpy as np

    from paper_2310_03567_b200 import _lib
    from paper_2310_03567_b200.render import Camera, brute_force_render

    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(_lib.NativeUnavailable):
        brute_force_render(np.zeros((1, 3), np.float32), np.zeros(1, np.uint32),
                           Camera((0.5, 0.5, -1.0), (0.5, 0.5, 0.5)))


def test_no_cpu_fallback_tree_creation():
    from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, _lib

    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    arena = Arena(1 << 20)
    with pytest.raises(_lib.NativeUnavailable):
        Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 16))


def test_status_codes_map_to_reference_exceptions():
    from paper_2310_03567_b200 import BacklogOverflow, OutOfArena, SpillOverflow, _lib

    for code, exc in ((1, OutOfArena), (2, SpillOverflow), (3, BacklogOverflow)):
        with pytest.raises(exc):
            _lib.check(code)
    assert issubclass(OutOfArena, MemoryError)
