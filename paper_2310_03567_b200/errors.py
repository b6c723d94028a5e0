"""Exception types of the LOD update path (reference: lodstream/errors.py:1-19).

Resource exhaustion (arena, spill, backlog) is fatal: the tree may be left
partially updated.  The C ABI reports these as LOD_E_OUT_OF_ARENA,
LOD_E_SPILL_OVERFLOW and LOD_E_BACKLOG_OVERFLOW; ``_lib.check`` maps them here.
"""
from __future__ import annotations


class OutOfArena(MemoryError):
    """Arena capacity exhausted.  The arena never frees, so this is fatal."""


class SpillOverflow(RuntimeError):
    """Spill buffer exceeded its configured capacity during a split."""


class BacklogOverflow(RuntimeError):
    """Voxel backlog exceeded its configured capacity during sampling."""
