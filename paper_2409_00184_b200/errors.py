"""Error hierarchy of the B200 path.

The names and base classes are the reference's (splinecast errors.py:12-25)
so callers catching them keep working; libafam status codes map onto them
in _lib.check (include/afam.h: 1 missing block, 2 format, 3 capacity,
4 bad value).
"""

from __future__ import annotations

__all__ = ["FormatError", "PartitionError", "CapacityError", "MissingBlockError"]


class FormatError(ValueError):
    """Bytes on disk (.mfa, manifest.json, trajectory) disagree with FORMAT.md."""


class PartitionError(ValueError):
    """Requested LOD hierarchy cannot be cut from the given lattice."""


class CapacityError(RuntimeError):
    """Block cache / device slots cannot hold the frame's visible set."""


class MissingBlockError(RuntimeError):
    """A sample fell into a finest cell that no resident block owns."""
