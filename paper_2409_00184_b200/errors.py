"""Error hierarchy of the B200 path.

These are the reference's exception types (splinecast errors.py:12-25):
when the reference package is importable (the drop-in setting of
INTEGRATION.md, where reference callers such as cli.py:345-351,
service.py:255 and tests/test_render.py:360 catch
``splinecast.errors.*``), the classes ARE the reference's, re-exported;
otherwise classes with the same names and bases stand in.  libafam status
codes map onto them in _lib.check (include/afam.h: 1 missing block,
2 format, 3 capacity, 4 bad value).
"""

from __future__ import annotations

__all__ = ["FormatError", "PartitionError", "CapacityError", "MissingBlockError", "REFERENCE_CLASSES"]

try:  # the drop-in: raise the caller's own exception types
    from splinecast.errors import CapacityError, FormatError, MissingBlockError, PartitionError

    REFERENCE_CLASSES = True
except ImportError:
    REFERENCE_CLASSES = False

    class FormatError(ValueError):
        """Bytes on disk (.mfa, manifest.json, trajectory) disagree with FORMAT.md."""

    class PartitionError(ValueError):
        """Requested LOD hierarchy cannot be cut from the given lattice."""

    class CapacityError(RuntimeError):
        """Block cache / device slots cannot hold the frame's visible set."""

    class MissingBlockError(RuntimeError):
        """A sample fell into a finest cell that no resident block owns."""
