"""ctypes front-end of the float64 CPU oracle (oracle/afam_oracle.c).

TEST INFRASTRUCTURE ONLY.  This module is the parity checker for the B200
path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import it; the product package never does.

It takes duck-typed inputs (anything shaped like the reference's
PointOfView / TransferFunction / RenderParams / MicroModel / LODManifest),
so the same checker can be fed reference objects (to pin it against the
unmodified reference, tests/golden/gen_golden.py) and product objects (to
check the CUDA path).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libafam_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc only, no CUDA)."""
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < (_HERE / "afam_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


class _Block(C.Structure):
    _fields_ = [
        ("ctrl", C.c_void_p),
        ("knots", C.c_void_p),
        ("lo", C.c_double * 3),
        ("hi", C.c_double * 3),
        ("ncp", C.c_int),
        ("deg", C.c_int),
    ]


class _Frame(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3),
        ("f", C.c_double * 3),
        ("r", C.c_double * 3),
        ("u", C.c_double * 3),
        ("tan_x", C.c_double),
        ("tan_y", C.c_double),
        ("width", C.c_int),
        ("height", C.c_int),
        ("row0", C.c_int),
        ("row1", C.c_int),
        ("sd", C.c_double),
        ("power", C.c_double),
        ("o_max", C.c_double),
        ("near_", C.c_double),
        ("ambient", C.c_double),
        ("diffuse", C.c_double),
        ("specular", C.c_double),
        ("shininess", C.c_double),
        ("color_pts", C.c_void_p),
        ("ncolor", C.c_int),
        ("opac_pts", C.c_void_p),
        ("nopac", C.c_int),
        ("dom_lo", C.c_double),
        ("dom_hi", C.c_double),
    ]


class _Stats(C.Structure):
    _fields_ = [("samples", C.c_int64), ("missing_key", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(_LIB_PATH))
        _lib.afo_find_span.restype = C.c_int
        _lib.afo_find_span.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double]
        _lib.afo_basis.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]
        _lib.afo_basis_ders.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        _lib.afo_eval_points.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.afo_decode_grid.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib.afo_lod_for_distance.restype = C.c_int
        _lib.afo_lod_for_distance.argtypes = [C.c_double, C.c_int, C.c_void_p, C.c_int]
        _lib.afo_select_visible.restype = C.c_int
        _lib.afo_select_visible.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                            C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _lib.afo_owner_grid.restype = C.c_int
        _lib.afo_owner_grid.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _lib.afo_render.restype = C.c_int
        _lib.afo_render.argtypes = [C.POINTER(_Frame), C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.POINTER(_Stats), C.c_int]
        _lib.afo_max_threads.restype = C.c_int
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ctrl_xfast(control) -> np.ndarray:
    """(ncp,ncp,ncp) [ix,iy,iz] -> flat float32, x fastest (FORMAT.md:57-61)."""
    c = np.asarray(control, dtype=np.float32)
    return np.ascontiguousarray(c.ravel(order="F"))


def max_threads() -> int:
    return int(lib().afo_max_threads())


# ---------------------------------------------------------------- numerics
def find_span(knots, ncp: int, degree: int, u: float) -> int:
    kv = _f64(knots)
    return int(lib().afo_find_span(_ptr(kv), kv.size, ncp, degree, float(u)))


def basis(knots, degree: int, span: int, u: float, derivatives: bool = False):
    kv = _f64(knots)
    n = np.zeros(degree + 1)
    if derivatives:
        d = np.zeros(degree + 1)
        lib().afo_basis_ders(_ptr(kv), degree, span, float(u), _ptr(n), _ptr(d))
        return n, d
    lib().afo_basis(_ptr(kv), degree, span, float(u), _ptr(n))
    return n


def eval_points(control, degree: int, u, knots=None, gradient: bool = True):
    """bspline.evaluate_points[_with_gradient] (bspline.py:206-229), float64."""
    c = _ctrl_xfast(control)
    ncp = int(round(c.size ** (1.0 / 3.0)))
    uu = _f64(np.atleast_2d(np.asarray(u, dtype=np.float64)))
    n = uu.shape[0]
    val = np.zeros(n)
    grad = np.zeros((n, 3)) if gradient else None
    kv = None if knots is None else _f64(np.asarray(knots, dtype=np.float64).reshape(3, -1))
    lib().afo_eval_points(_ptr(c), ncp, degree, None if kv is None else _ptr(kv), n, _ptr(uu), _ptr(val),
                          None if grad is None else _ptr(grad))
    return (val, grad) if gradient else val


def decode_grid(control, degree: int, m: int) -> np.ndarray:
    """MicroModel.decode_grid((m,m,m)) (model.py:89-93); returns [i,j,k] float64."""
    c = _ctrl_xfast(control)
    ncp = int(round(c.size ** (1.0 / 3.0)))
    out = np.zeros(m * m * m)
    lib().afo_decode_grid(_ptr(c), ncp, degree, m, _ptr(out))
    return out.reshape((m, m, m), order="F")


# ---------------------------------------------------------------- camera
def camera_basis(pov):
    """PointOfView.basis() (render.py:68-73) on the host with numpy."""
    f = np.asarray(pov.direction, dtype=np.float64)
    r = np.cross(f, np.asarray(pov.up, dtype=np.float64))
    r = r / np.linalg.norm(r)
    return f, r, np.cross(r, f)


def lod_for_distance(d: float, levels: int, ranges=None) -> int:
    rr = None if ranges is None else _f64(ranges)
    return int(lib().afo_lod_for_distance(float(d), levels, None if rr is None else _ptr(rr),
                                          0 if rr is None else rr.size))


def _manifest_tables(manifest):
    levels = int(manifest.levels)
    coarsest = int(manifest.finest_blocks_per_axis) >> (levels - 1)
    bpa = np.array([coarsest * 2 ** (levels - l) for l in range(1, levels + 1)], dtype=np.int32)
    tabs = []
    for l in range(1, levels + 1):
        b = int(bpa[l - 1])
        t = np.zeros((b, b, b, 6))
        for addr, entry in manifest.entries.items():
            if addr.lod == l:
                i, j, k = addr.ijk
                t[i, j, k] = np.asarray(entry.extent, dtype=np.float64).reshape(3, 2).ravel()
        tabs.append(np.ascontiguousarray(t))
    return levels, bpa, tabs


def select_visible(pov, manifest, aspect: float = 1.0, near: float = 1e-3, ranges=None):
    """render.select_visible (render.py:281-320) -> sorted list of (lod, i, j, k)."""
    levels, bpa, tabs = _manifest_tables(manifest)
    ptrs = (C.c_void_p * levels)(*[t.ctypes.data for t in tabs])
    f, r, u = camera_basis(pov)
    pos = _f64(pov.position)
    tan_y = math.tan(math.radians(pov.fov_y) / 2.0)
    rr = None if ranges is None else _f64(ranges)
    cap = int(sum(int(b) ** 3 for b in bpa))
    out = np.zeros((cap, 4), dtype=np.int32)
    n = lib().afo_select_visible(levels, _ptr(bpa), C.cast(ptrs, C.c_void_p), _ptr(pos), _ptr(_f64(f)),
                                 _ptr(_f64(r)), _ptr(_f64(u)), tan_y, float(aspect), float(near),
                                 None if rr is None else _ptr(rr), 0 if rr is None else rr.size,
                                 _ptr(out), cap)
    return [tuple(int(v) for v in row) for row in out[:n]]


# ---------------------------------------------------------------- render
def _blocks(blocks_sorted):
    keep = []
    arr = (_Block * max(1, len(blocks_sorted)))()
    for i, blk in enumerate(blocks_sorted):
        c = _ctrl_xfast(blk.control)
        kv = _f64(np.asarray(blk.knots, dtype=np.float32).astype(np.float64))
        ext = np.asarray(blk.extent, dtype=np.float64).reshape(3, 2)
        keep += [c, kv]
        arr[i].ctrl = c.ctypes.data
        arr[i].knots = kv.ctypes.data
        for a in range(3):
            arr[i].lo[a] = ext[a, 0]
            arr[i].hi[a] = ext[a, 1]
        arr[i].ncp = int(np.asarray(blk.control).shape[0])
        arr[i].deg = int(blk.degree)
    return arr, keep


def render(pov, blocks: dict, tf, params, rows=None, nthreads: int = 0, debug: bool = False):
    """render.render (render.py:398-466) in float64, one ray at a time.

    Returns (rgba (rows,W,4) uint8, info dict).  info has 'samples',
    'missing' ((step, ray) of the first sample in an uncovered finest cell,
    or None) and, with debug, per-ray 'nsamp' and 'ohash'.
    """
    addrs = sorted(blocks)
    arr, keep = _blocks([blocks[a] for a in addrs])
    W, H = int(params.width), int(params.height)
    r0, r1 = (0, H) if rows is None else (int(rows[0]), int(rows[1]))
    f, r, u = camera_basis(pov)
    tan_y = math.tan(math.radians(pov.fov_y) / 2.0)
    fr = _Frame()
    for a in range(3):
        fr.origin[a] = float(np.asarray(pov.position, dtype=np.float64)[a])
        fr.f[a], fr.r[a], fr.u[a] = float(f[a]), float(r[a]), float(u[a])
    fr.tan_y = tan_y
    fr.tan_x = tan_y * (W / H)
    fr.width, fr.height, fr.row0, fr.row1 = W, H, r0, r1
    sd = float(params.sample_distance)
    ref = params.reference_step if params.reference_step is not None else sd
    fr.sd, fr.power, fr.o_max, fr.near_ = sd, sd / ref, float(params.o_max), float(params.near)
    fr.ambient, fr.diffuse = float(params.ambient), float(params.diffuse)
    fr.specular, fr.shininess = float(params.specular), float(params.shininess)
    cp = _f64(tf.color_points)
    op = _f64(tf.opacity_points)
    fr.color_pts, fr.ncolor = cp.ctypes.data, cp.shape[0]
    fr.opac_pts, fr.nopac = op.ctypes.data, op.shape[0]
    fr.dom_lo, fr.dom_hi = float(tf.domain[0]), float(tf.domain[1])
    nr = (r1 - r0) * W
    rgba = np.zeros((r1 - r0, W, 4), dtype=np.uint8)
    nsamp = np.zeros(nr, dtype=np.int32) if debug else None
    ohash = np.zeros(nr, dtype=np.uint64) if debug else None
    st = _Stats()
    lib().afo_render(C.byref(fr), C.cast(arr, C.c_void_p), len(addrs), _ptr(rgba),
                     None if nsamp is None else _ptr(nsamp), None if ohash is None else _ptr(ohash),
                     C.byref(st), int(nthreads))
    missing = None
    if st.missing_key >= 0:
        missing = (int(st.missing_key) >> 32, int(st.missing_key) & 0xFFFFFFFF)
    info = {"samples": int(st.samples), "missing": missing}
    if debug:
        info["nsamp"] = nsamp
        info["ohash"] = ohash
    del keep
    return rgba, info


def owner_grid(blocks_sorted):
    arr, keep = _blocks(blocks_sorted)
    cells = lib().afo_owner_grid(C.cast(arr, C.c_void_p), len(blocks_sorted), None, 0)
    g = np.zeros(cells ** 3, dtype=np.int32)
    lib().afo_owner_grid(C.cast(arr, C.c_void_p), len(blocks_sorted), _ptr(g), cells)
    del keep
    return cells, g.reshape(cells, cells, cells)


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """metrics.psnr semantics (metrics.py:38-49): RGB only, alpha excluded, unit peak."""
    x = np.asarray(a, dtype=np.float64)[..., :3] / 255.0
    y = np.asarray(b, dtype=np.float64)[..., :3] / 255.0
    mse = float(np.mean((x - y) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)
