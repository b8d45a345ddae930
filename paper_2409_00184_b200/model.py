"""Micro-model type and the .mfa byte codec (host side).

MicroModel mirrors the reference's frozen dataclass (reference
model.py:27-93) field for field; its decode hooks (values_at,
gradients_at, query_*, decode_grid) run on the GPU through the scratch
device store.  serialize / deserialize implement FORMAT.md:16-70:

    [u8 degree][3 x (ncp+degree) float32 knots t1..][ncp^3 float32, x fastest]

and raise FormatError exactly where the reference does (model.py:121-133).
Least-squares fitting (model.fit) is encoder-side and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import FormatError

__all__ = ["MicroModel", "serialized_size", "serialize", "deserialize", "parse_header"]


def serialized_size(ncp: int, degree: int) -> int:
    """Bytes of one .mfa file: 1 + ((ncp + degree)*3 + ncp^3)*4."""
    return 1 + 4 * (3 * (ncp + degree) + ncp ** 3)


@dataclass(frozen=True, eq=False)
class MicroModel:
    degree: int
    knots: np.ndarray     # (3, ncp+degree+1) float32 full clamped vectors
    control: np.ndarray   # (ncp, ncp, ncp) float32, [ix, iy, iz]
    extent: np.ndarray    # (3, 2) float64 box in [-1, 1]^3
    lod: int

    def __post_init__(self):
        ctrl = np.asarray(self.control, dtype=np.float32)
        n = ctrl.shape[0] if ctrl.ndim == 3 else -1
        if ctrl.ndim != 3 or ctrl.shape != (n, n, n):
            raise ValueError(f"control grid must be cubic, got {ctrl.shape}")
        kv = np.asarray(self.knots, dtype=np.float32)
        if kv.shape != (3, n + self.degree + 1):
            raise ValueError(f"knot vectors must be (3, {n + self.degree + 1}), got {kv.shape}")
        if not np.isfinite(ctrl).all():
            raise ValueError("non-finite control points")
        ext = np.asarray(self.extent, dtype=np.float64).reshape(3, 2)
        if (ext[:, 1] <= ext[:, 0]).any():
            raise ValueError("degenerate extent")
        object.__setattr__(self, "control", ctrl)
        object.__setattr__(self, "knots", kv)
        object.__setattr__(self, "extent", ext)

    @property
    def ncp(self) -> int:
        return int(self.control.shape[0])

    @property
    def nbytes(self) -> int:
        return serialized_size(self.ncp, self.degree)

    def params_for(self, points) -> np.ndarray:
        lo = self.extent[:, 0]
        return np.clip((np.atleast_2d(points) - lo) / (self.extent[:, 1] - lo), 0.0, 1.0)

    # --- decode hooks: B200 kernels (K1 / K3) ------------------------------
    def _resident(self):
        from .device import as_device_blocks

        store, (slot,) = as_device_blocks([self])
        return store, slot

    def query_value(self, u) -> np.ndarray:
        from .bspline import eval_device

        store, slot = self._resident()
        return eval_device(store, slot, u, gradient=False, param=True)

    def query_gradient(self, u) -> np.ndarray:
        from .bspline import eval_device

        store, slot = self._resident()
        _, g = eval_device(store, slot, u, gradient=True, param=True)
        return g / (self.extent[:, 1] - self.extent[:, 0])

    def values_at(self, points) -> np.ndarray:
        from .bspline import eval_device

        store, slot = self._resident()
        return eval_device(store, slot, points, gradient=False)

    def gradients_at(self, points) -> np.ndarray:
        from .bspline import eval_device

        store, slot = self._resident()
        return eval_device(store, slot, points, gradient=True)[1]

    def decode_grid(self, dims) -> np.ndarray:
        from .bspline import decode_block

        store, slot = self._resident()
        return decode_block(store, slot, dims)


def serialize(model) -> bytes:
    if not 0 <= model.degree <= 255:
        raise FormatError(f"degree {model.degree} does not fit the header byte")
    kv = np.asarray(model.knots, dtype="<f4")
    body = [kv[a, 1:].tobytes() for a in range(3)]
    ctrl = np.asarray(model.control, dtype="<f4").ravel(order="F").tobytes()
    return bytes([int(model.degree)]) + b"".join(body) + ctrl


def parse_header(data, ncp: int) -> int:
    """Validate an .mfa image against its manifest ncp; returns the degree."""
    if len(data) < 1:
        raise FormatError("empty micro-model byte string")
    deg = int(data[0])
    if deg >= ncp:
        raise FormatError(f"degree byte {deg} >= ncp {ncp}")
    want = serialized_size(ncp, deg)
    if len(data) != want:
        raise FormatError(f"micro-model length mismatch: expected {want} bytes "
                          f"for ncp={ncp}, degree={deg}, found {len(data)}")
    return deg


def deserialize(data: bytes, ncp: int, extent, lod: int) -> MicroModel:
    deg = parse_header(data, ncp)
    m = ncp + deg
    raw = np.frombuffer(data, dtype="<f4", count=3 * m, offset=1).reshape(3, m)
    knots = np.zeros((3, m + 1), dtype=np.float32)
    knots[:, 1:] = raw
    ctrl = np.frombuffer(data, dtype="<f4", count=ncp ** 3, offset=1 + 12 * m)
    return MicroModel(degree=deg, knots=knots, control=ctrl.reshape((ncp,) * 3, order="F").copy(),
                      extent=np.asarray(extent, dtype=np.float64), lod=lod)
