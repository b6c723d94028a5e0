"""The SIM disk feed (io.py:60-92, 218-290, 340-413): file layout, the native
O_DIRECT reader thread's batches in file order, truncated / empty files.
CPU only (the reader needs no GPU); the GPU test streams a file into a tree."""
import os

import numpy as np
import pytest

from paper_2310_03567_b200 import _lib, ingest, synth


def _lib_ok():
    try:
        _lib.load()
        return True
    except Exception:
        return False


pytestmark = pytest.mark.skipif(not _lib_ok(), reason="library not built")


def test_sim_layout_matches_the_record_layout(tmp_path):
    xyz, rgba = synth.gen_uniform(1000, 1)
    p = tmp_path / "a.sim"
    ingest.write_sim(p, xyz, rgba)
    rec = np.fromfile(p, ingest.SIM_DTYPE)  # the reference's structured view (io.py:38-40)
    assert np.array_equal(rec["x"], xyz[:, 0]) and np.array_equal(rec["z"], xyz[:, 2])
    assert np.array_equal(rec["r"], (rgba & 0xFF).astype(np.uint8))
    assert np.array_equal(rec["a"], (rgba >> 24).astype(np.uint8))
    x2, c2 = ingest.read_sim(p)
    assert np.array_equal(x2, xyz) and np.array_equal(c2, rgba)


@pytest.mark.parametrize("readers", [1, 6])
@pytest.mark.parametrize("n,batch", [(1_000_000, 65_536), (300_000, 1_048_576), (256, 256), (5000, 512)])
def test_reader_threads_return_every_batch_in_order(tmp_path, monkeypatch, n, batch, readers):
    """1 reader thread, or 6 reading batches concurrently (LOD_SIM_READERS)."""
    monkeypatch.setenv("LOD_SIM_READERS", str(readers))
    xyz, rgba = synth.gen_surface(n, 2)
    p = tmp_path / "b.sim"
    ingest.write_sim(p, xyz, rgba)
    src = ingest.SimSource(p, batch, slots=8)
    got = [b.copy() for b in src]
    info = src.info()
    src.close()
    assert [len(b) for b in got] == [min(batch, n - i) for i in range(0, n, batch)]
    rec = np.concatenate(got)
    assert np.array_equal(rec[:, :3].view(np.float32), xyz) and np.array_equal(rec[:, 3], rgba)
    assert info["bytes_read"] == info["file_bytes"] == 16 * n


def test_truncated_and_empty_files_are_refused(tmp_path):
    p = tmp_path / "t.sim"
    p.write_bytes(b"\0" * 40)  # 2.5 records (io.py: Truncated)
    with pytest.raises(ValueError):
        ingest.SimSource(p, 256)
    e = tmp_path / "e.sim"
    e.write_bytes(b"")  # io.py: EmptyFile
    with pytest.raises(ValueError):
        ingest.SimSource(e, 256)
    with pytest.raises(ValueError):
        ingest.SimSource(p, 100)  # 1600-byte batches break O_DIRECT alignment


@pytest.mark.gpu
def test_stream_sim_equals_inserting_the_batches(gpu, tmp_path):
    """stream_sim (native reader -> staged DMA -> insert_records, render per
    frame) builds the same tree as insert_batch over the same batches."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from common import assert_same_state, make_product, product_state

    from paper_2310_03567_b200 import insert_batch
    from paper_2310_03567_b200.render import Camera

    params = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=2 << 30, chunk_capacity=1000, grid_res=128,
                  leaf_threshold=50_000, max_depth=20, backlog_capacity=64_000_000, spill_capacity=100_000_000)
    parts = [synth.gen_surface(1_048_576, 40 + i) for i in range(6)]
    xyz = np.concatenate([x for x, _ in parts])
    rgba = np.concatenate([c for _, c in parts])
    p = tmp_path / "s.sim"
    ingest.write_sim(p, xyz, rgba)
    a, sa = make_product(params)
    cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), width=640, height=480)
    out = ingest.stream_sim(a, p, sa, batch_size=1_048_576, camera=cam)
    assert out["points"] == len(rgba) and out["batches"] == 6 and out["frames"] == 6
    b, sb = make_product(params)
    for x, c in parts:
        insert_batch(b, x, c, sb)
    assert_same_state(product_state(a), product_state(b), chunk_ids=False, label="stream_sim")
    assert sa.stats.voxels_created == sb.stats.voxels_created
