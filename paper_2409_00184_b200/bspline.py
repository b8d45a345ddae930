"""B-spline decode entry points of the reference's bspline module, on B200.

Drop-in for reference bspline.py:162-229 (evaluate_points,
evaluate_points_with_gradient, decode_tensor_product): the arithmetic runs
in libafam's K1 (point decode) and K3 (grid decode) kernels.  Results are
float32 on device (float64 for ill-conditioned grids, see include/afam.h
AFAM_SLOT_FP64) and returned as float64 arrays, within the 1e-5 x range
gate of BASELINE.json's north_star.  Knot vectors travel as float32 (the
.mfa storage type, FORMAT.md:22-30).

The least-squares fit (bspline.py:109-159) is encoder-side and out of
scope; clamped_knots is kept because callers build default knots with it.
"""

from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np

from . import _lib
from .device import as_device_blocks, stream_handle

__all__ = ["clamped_knots", "evaluate_points", "evaluate_points_with_gradient", "decode_tensor_product",
           "eval_device", "decode_slots"]


def clamped_knots(ncp: int, degree: int) -> np.ndarray:
    """Full clamped uniform knot vector on [0, 1], length ncp+degree+1."""
    if degree < 1:
        raise ValueError(f"degree must be >= 1, got {degree}")
    if ncp < degree + 1:
        raise ValueError(f"ncp must be >= degree+1 ({degree + 1}), got {ncp}")
    nspan = ncp - degree
    inner = np.arange(1, nspan, dtype=np.float64) / nspan
    return np.r_[np.zeros(degree + 1), inner, np.ones(degree + 1)]


def _torch():
    import torch

    return torch


def eval_device(store, slots, points, gradient: bool = True, param: bool = False, out_f64: bool = True):
    """K1 on resident slots: `slots` is one slot id or an int array (n,).
    Returns values (n,) [and gradients (n, 3)] as float64 numpy arrays
    (device output float64 unless out_f64=False)."""
    torch = _torch()
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, dtype=np.float64)))
    if pts.shape[-1] != 3:
        raise ValueError(f"points must have shape (n, 3), got {pts.shape}")
    n = pts.shape[0]
    dev = torch.device("cuda", store.device)
    odt = torch.float64 if out_f64 else torch.float32
    d_pts = torch.from_numpy(pts).to(dev, non_blocking=False)
    d_val = torch.empty(n, dtype=odt, device=dev)
    d_grad = torch.empty((n, 3), dtype=odt, device=dev) if gradient else None
    one_slot, d_slots = 0, None
    if np.ndim(slots) == 0:
        one_slot = int(slots)
    else:
        d_slots = torch.from_numpy(np.ascontiguousarray(slots, dtype=np.int32)).to(dev)
    flags = (_lib.AFAM_EVAL_PARAM if param else 0) | (_lib.AFAM_EVAL_OUT_F64 if out_f64 else 0)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().afam_eval_points(
            store.handle, None if d_slots is None else C.c_void_p(d_slots.data_ptr()), one_slot,
            C.c_void_p(d_pts.data_ptr()), n, C.c_void_p(d_val.data_ptr()),
            None if d_grad is None else C.c_void_p(d_grad.data_ptr()), flags, C.c_void_p(stream_handle(None, dev))))
        val = d_val.cpu().numpy().astype(np.float64)
        if not gradient:
            return val
        return val, d_grad.cpu().numpy().astype(np.float64)


DECODE_PATHS = {"auto": 0, "cuda_cores": 1, "tensor_cores": 2}


def decode_slots(store, slots, m: int, path: str = "auto", info: dict | None = None) -> np.ndarray:
    """K3 on resident slots -> (nblk, m, m, m) float64 array indexed [b, i, j, k].
    path: "auto" | "cuda_cores" | "tensor_cores" (afam_decode_grid_ex); info,
    if given, receives {"tensor_core_blocks": n}."""
    torch = _torch()
    if path not in DECODE_PATHS:
        raise ValueError(f"unknown decode path {path!r} (use {', '.join(DECODE_PATHS)})")
    slots = np.ascontiguousarray(slots, dtype=np.int32)
    dev = torch.device("cuda", store.device)
    out = torch.empty((len(slots), m, m, m), dtype=torch.float32, device=dev)
    ntc = C.c_int32(0)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().afam_decode_grid_ex(store.handle, slots.ctypes.data_as(C.c_void_p), len(slots), int(m),
                                                  C.c_void_p(out.data_ptr()), DECODE_PATHS[path], C.byref(ntc),
                                                  C.c_void_p(stream_handle(None, dev))))
        host = out.cpu().numpy()
    if info is not None:
        info["tensor_core_blocks"] = int(ntc.value)
    # device layout is x fastest within a block: [b][k][j][i]
    return np.ascontiguousarray(host.transpose(0, 3, 2, 1)).astype(np.float64)


def _as_model(coeff, degree, knots):
    c = np.asarray(coeff)
    ncp = c.shape[0]
    if c.ndim != 3 or c.shape[1] != ncp or c.shape[2] != ncp:
        raise ValueError("coefficient grid must be cubic (isotropic ncp)")
    if knots is None:
        kv = np.repeat(clamped_knots(ncp, degree)[None, :], 3, axis=0)
    else:
        kv = np.stack([np.asarray(k, dtype=np.float64) for k in knots])
    return _GridModel(c, kv.astype(np.float32), int(degree))


class _GridModel:
    """A bare coefficient grid posing as a model on the unit extent (weak-referenceable,
    so the scratch store can tell a recycled id() from the same object)."""

    __slots__ = ("control", "knots", "degree", "extent", "lod", "__weakref__")

    def __init__(self, control, knots, degree):
        self.control, self.knots, self.degree = control, knots, degree
        self.extent = np.array([[0.0, 1.0]] * 3)
        self.lod = 1


def evaluate_points(coeff, degree: int, u, knots=None) -> np.ndarray:
    """Spline values at parameters u (n, 3) (reference bspline.py:206-214)."""
    store, (slot,) = as_device_blocks([_as_model(coeff, degree, knots)])
    return eval_device(store, slot, u, gradient=False, param=True)


def evaluate_points_with_gradient(coeff, degree: int, u, knots=None):
    """Values and parameter-space gradients (reference bspline.py:217-229)."""
    store, (slot,) = as_device_blocks([_as_model(coeff, degree, knots)])
    return eval_device(store, slot, u, gradient=True, param=True)


def decode_tensor_product(coeff, degree: int, dims) -> np.ndarray:
    """Decode onto the uniform dims lattice (reference bspline.py:162-172)."""
    store, (slot,) = as_device_blocks([_as_model(coeff, degree, None)])
    return decode_block(store, slot, dims)


def decode_block(store, slot: int, dims) -> np.ndarray:
    """One resident block on the uniform dims lattice, float64 [i, j, k].
    Cubic dims take K3 (afam_decode_grid_ex); other shapes evaluate the
    lattice parameters linspace(0, 1, d) per axis with K1 (param mode), the
    reference's u grid (bspline.py:117)."""
    d = tuple(int(v) for v in np.broadcast_to(np.asarray(dims), (3,)))
    if min(d) < 1:
        raise ValueError(f"decode dims must be positive, got {d}")
    if d[0] == d[1] == d[2] and d[0] >= 2:
        return decode_slots(store, [slot], d[0])[0]
    axes = [np.linspace(0.0, 1.0, n) for n in d]
    u = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    return eval_device(store, int(slot), u, gradient=False, param=True).reshape(d)


