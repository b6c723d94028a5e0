"""B200-native incremental point-cloud LOD construction (arXiv 2310.03567).

Drop-in for the reference package ``lodstream``'s hot path: the same public
names (``Arena``, ``ChunkPool``, ``CubeBounds``, ``Octree``, ``UpdateConfig``,
``UpdateState``, ``cubify``, ``insert_batch``, ``run_frame_updates``; plus
``render.rasterize`` / ``render.brute_force_render``), backed by hand-written
sm_100a CUDA kernels in ``_lodb200.so`` (C ABI: include/lod_b200.h).  There is
no CPU fallback: without the library or a CUDA device the entry points raise.
"""
from .errors import BacklogOverflow, OutOfArena, SpillOverflow
from .octree import CubeBounds, Octree, cubify
from .store import Arena, ChunkPool
from .update import BatchDelta, UpdateConfig, UpdateState, insert_batch, run_frame_updates, wait_settled

__version__ = "0.1.0"

__all__ = [
    "Arena",
    "ChunkPool",
    "CubeBounds",
    "Octree",
    "BatchDelta",
    "UpdateConfig",
    "UpdateState",
    "cubify",
    "insert_batch",
    "run_frame_updates",
    "wait_settled",
    "OutOfArena",
    "SpillOverflow",
    "BacklogOverflow",
    "__version__",
]
