"""Camera, transfer function, visible-set selection and the B200 ray caster.

Drop-in for the reference's render module (reference render.py):
PointOfView / TransferFunction / RenderParams / Frame keep the reference's
fields, validation and JSON forms; select_visible runs in native C++
(libafam afam_select_visible, bit-exact with render.py:281-320) and
render() runs the fused K2 ray-march kernel (afam_render) over blocks
resident in HBM.  There is no CPU fallback: blocks must be spline
micro-models (MicroModel or DeviceBlock).
"""

from __future__ import annotations

import ctypes as C
import json
import math
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import MissingBlockError
from .partition import BlockAddress

__all__ = ["PointOfView", "TransferFunction", "RenderParams", "Frame", "default_lod_ranges", "lod_for_distance",
           "select_visible", "render", "render_part", "NativeManifest", "camera_setup"]

DOMAIN_LO, DOMAIN_HI = -1.0, 1.0


def pov_basis(pov):
    """(forward, right, up) of any pov-like object with the reference's numpy
    op order (render.py:68-73); direction is used as stored (already unit).
    Cached on PointOfView objects (immutable), which the replay loop asks
    for several times per frame."""
    cached = getattr(pov, "_afam_basis", None)
    if cached is not None:
        return cached
    fwd = np.asarray(pov.direction, dtype=np.float64)
    right = np.cross(fwd, np.asarray(pov.up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    out = (fwd, right, np.cross(right, fwd))
    if isinstance(pov, PointOfView):
        object.__setattr__(pov, "_afam_basis", out)
    return out


@dataclass(frozen=True, eq=False)
class PointOfView:
    position: np.ndarray
    direction: np.ndarray
    up: np.ndarray
    fov_y: float = 45.0

    def __post_init__(self):
        pos = np.asarray(self.position, dtype=np.float64).reshape(3)
        d = np.asarray(self.direction, dtype=np.float64).reshape(3)
        up = np.asarray(self.up, dtype=np.float64).reshape(3)
        n = np.linalg.norm(d)
        if n < 1e-12:
            raise ValueError("view direction has zero length")
        d = d / n
        if np.linalg.norm(np.cross(d, up)) < 1e-9:
            raise ValueError("up vector is parallel to the view direction")
        if not 0.0 < self.fov_y < 180.0:
            raise ValueError(f"fov_y {self.fov_y} out of (0, 180)")
        object.__setattr__(self, "position", pos)
        object.__setattr__(self, "direction", d)
        object.__setattr__(self, "up", up)

    def basis(self):
        return pov_basis(self)

    def to_json(self) -> dict:
        return {"pos": self.position.tolist(), "dir": self.direction.tolist(), "up": self.up.tolist(),
                "fov_y": self.fov_y}

    @classmethod
    def from_json(cls, obj: dict) -> "PointOfView":
        return cls(np.asarray(obj["pos"], dtype=np.float64), np.asarray(obj["dir"], dtype=np.float64),
                   np.asarray(obj["up"], dtype=np.float64), float(obj.get("fov_y", 45.0)))


@dataclass(frozen=True, eq=False)
class TransferFunction:
    color_points: np.ndarray    # (n, 4): scalar, r, g, b
    opacity_points: np.ndarray  # (m, 2): scalar, alpha
    domain: tuple = (0.0, 1.0)

    def __post_init__(self):
        cp = np.asarray(self.color_points, dtype=np.float64).reshape(-1, 4)
        op = np.asarray(self.opacity_points, dtype=np.float64).reshape(-1, 2)
        for pts, what in ((cp, "color"), (op, "opacity")):
            if pts.shape[0] < 1:
                raise ValueError(f"need at least one {what} control point")
            if (np.diff(pts[:, 0]) <= 0).any():
                raise ValueError(f"{what} control scalars must strictly increase")
            if pts[:, 1:].min() < 0 or pts[:, 1:].max() > 1:
                raise ValueError(f"{what} values must lie in [0,1]")
        lo, hi = float(self.domain[0]), float(self.domain[1])
        if not lo < hi:
            raise ValueError("degenerate domain")
        object.__setattr__(self, "color_points", cp)
        object.__setattr__(self, "opacity_points", op)
        object.__setattr__(self, "domain", (lo, hi))

    def color_at(self, values) -> np.ndarray:
        v = np.clip(values, *self.domain)
        xs = self.color_points[:, 0]
        return np.stack([np.interp(v, xs, self.color_points[:, c]) for c in (1, 2, 3)], axis=-1)

    def opacity_at(self, values) -> np.ndarray:
        v = np.clip(values, *self.domain)
        return np.interp(v, self.opacity_points[:, 0], self.opacity_points[:, 1])

    def to_json(self) -> dict:
        return {"domain": list(self.domain), "color": self.color_points.tolist(),
                "opacity": self.opacity_points.tolist()}

    @classmethod
    def from_json(cls, obj: dict) -> "TransferFunction":
        return cls(np.asarray(obj["color"], dtype=np.float64), np.asarray(obj["opacity"], dtype=np.float64),
                   tuple(obj.get("domain", (0.0, 1.0))))

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_json(), indent=2))

    @classmethod
    def load(cls, path) -> "TransferFunction":
        return cls.from_json(json.loads(Path(path).read_text()))

    @classmethod
    def ml_preset(cls) -> "TransferFunction":
        """The reference's `ml` preset (render.py:148-165)."""
        color = [[0.00, 0.10, 0.15, 0.60], [0.35, 0.20, 0.55, 0.85], [0.50, 0.95, 0.95, 0.90],
                 [0.65, 0.95, 0.55, 0.15], [1.00, 0.80, 0.20, 0.10]]
        alpha = [[0.00, 0.0], [0.38, 0.0], [0.50, 0.35], [0.62, 0.0], [1.00, 0.0]]
        return cls(np.array(color), np.array(alpha), (0.0, 1.0))


@dataclass
class RenderParams:
    width: int = 512
    height: int = 512
    sample_distance: float = 1e-3
    o_max: float = 0.99
    reference_step: float | None = None
    near: float = 1e-3
    ambient: float = 0.1
    diffuse: float = 0.7
    specular: float = 0.2
    shininess: float = 32.0
    lod_ranges: tuple | None = None

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("frame dimensions must be positive")
        if self.sample_distance <= 0:
            raise ValueError("sample distance must be positive")
        if not 0 < self.o_max <= 1:
            raise ValueError("o_max must be in (0, 1]")

    @property
    def aspect(self) -> float:
        return self.width / self.height


@dataclass
class Frame:
    width: int
    height: int
    rgba: np.ndarray  # (height, width, 4) uint8, row 0 at the top, premultiplied color

    def __post_init__(self):
        arr = np.asarray(self.rgba, dtype=np.uint8)
        if arr.shape != (self.height, self.width, 4):
            raise ValueError(f"rgba shape {arr.shape} != ({self.height}, {self.width}, 4)")
        self.rgba = arr

    def save_png(self, path) -> None:
        from PIL import Image

        Image.fromarray(self.rgba, mode="RGBA").save(Path(path), format="PNG")

    @classmethod
    def load_png(cls, path) -> "Frame":
        from PIL import Image

        img = Image.open(Path(path)).convert("RGBA")
        return cls(width=img.width, height=img.height, rgba=np.asarray(img, dtype=np.uint8))

    def to_png_bytes(self) -> bytes:
        """PNG of the frame (render.py:216-221): the image data is filtered and
        deflated on the GPU (png_bytes_gpu).  No CPU fallback: without a CUDA
        device this raises (the file-writing save_png is the host path)."""
        from . import _lib

        _lib.require_device()
        return png_bytes_gpu(self.rgba)


def png_bytes_gpu(rgba) -> bytes:
    """PNG bytes of an (H, W, 4) uint8 RGBA frame (host array or CUDA tensor):
    afam_png_deflate makes the zlib payload on the GPU, the host wraps the
    chunks (IHDR, IDAT, IEND with CRC-32)."""
    import struct
    import zlib

    import torch

    if isinstance(rgba, torch.Tensor) and rgba.is_cuda:
        d = rgba.contiguous()
    else:
        d = torch.from_numpy(np.ascontiguousarray(rgba, dtype=np.uint8)).cuda()
    H, W = int(d.shape[0]), int(d.shape[1])
    if d.shape[2] != 4 or d.dtype != torch.uint8:
        raise ValueError(f"expected (H, W, 4) uint8 RGBA, got {tuple(d.shape)} {d.dtype}")
    cap = int(((4 * W + 1) * 15 // 8 + 16) * H + 2048)
    out = torch.empty(cap, dtype=torch.uint8, device=d.device)
    nbytes, adler = C.c_uint64(), C.c_uint32()
    with torch.cuda.device(d.device):
        _lib.check(_lib.lib().afam_png_deflate(C.c_void_p(d.data_ptr()), W, H, C.c_void_p(out.data_ptr()), cap,
                                               C.byref(nbytes), C.byref(adler),
                                               C.c_void_p(torch.cuda.current_stream(d.device).cuda_stream)))
    body = out[: nbytes.value].cpu().numpy().tobytes()
    idat = b"\x78\x01" + body + struct.pack(">I", adler.value)

    def chunk(kind: bytes, data: bytes) -> bytes:
        return struct.pack(">I", len(data)) + kind + data + struct.pack(">I", zlib.crc32(kind + data) & 0xFFFFFFFF)

    ihdr = struct.pack(">IIBBBBB", W, H, 8, 6, 0, 0, 0)
    return b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", ihdr) + chunk(b"IDAT", idat) + chunk(b"IEND", b"")


# ------------------------------------------------------------- visibility
def default_lod_ranges(levels: int) -> np.ndarray:
    """Band upper bounds k*4.0/5.0, k = 1..levels-1 (render.py:249-253)."""
    return np.arange(1, levels) * 4.0 / 5.0


def lod_for_distance(d: float, levels: int, ranges=None) -> int:
    if d < 0:
        raise ValueError("distance must be nonnegative")
    bands = default_lod_ranges(levels) if ranges is None else np.asarray(ranges, dtype=np.float64)
    return int(np.searchsorted(bands, d, side="right")) + 1


class NativeManifest:
    """A manifest's level tables handed to libafam once (afam_manifest_create)."""

    def __init__(self, manifest):
        from .partition import level_tables

        bpa, tabs = level_tables(manifest)
        ptrs = (C.c_void_p * len(tabs))(*[t.ctypes.data for t in tabs])
        h = C.c_void_p()
        _lib.check(_lib.lib().afam_manifest_create(C.byref(h), len(tabs), bpa.ctypes.data_as(C.c_void_p),
                                                   C.cast(ptrs, C.c_void_p)))
        self._h = h
        self.levels = manifest.levels
        self.capacity = int(sum(int(b) ** 3 for b in bpa))
        self._out = np.zeros((self.capacity, 4), dtype=np.int32)
        # interned addresses: flat index off[lod-1] + (i*bpa + j)*bpa + k -> BlockAddress
        self._bpa = np.asarray(bpa, dtype=np.int64)
        self._off = np.concatenate([[0], np.cumsum(self._bpa ** 3)[:-1]]).astype(np.int64)
        self._addrs = [BlockAddress(l + 1, (i, j, k)) for l, b in enumerate(bpa.tolist())
                       for i in range(b) for j in range(b) for k in range(b)]

    def __del__(self):
        try:
            _lib.lib().afam_manifest_destroy(self._h)
        except Exception:
            pass

    def select(self, pov, aspect=1.0, near=1e-3, ranges=None):
        fwd, right, up = pov_basis(pov)
        f = np.ascontiguousarray(fwd, dtype=np.float64)
        r = np.ascontiguousarray(right, dtype=np.float64)
        u = np.ascontiguousarray(up, dtype=np.float64)
        pos = np.ascontiguousarray(pov.position, dtype=np.float64)
        rr = None if ranges is None else np.ascontiguousarray(ranges, dtype=np.float64)
        n = C.c_int32()
        _lib.check(_lib.lib().afam_select_visible(
            self._h, pos.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
            u.ctypes.data_as(C.c_void_p), math.tan(math.radians(pov.fov_y) / 2.0), float(aspect), float(near),
            None if rr is None else rr.ctypes.data_as(C.c_void_p), 0 if rr is None else rr.size,
            self._out.ctypes.data_as(C.c_void_p), self.capacity, C.byref(n)))
        q = self._out[: n.value].astype(np.int64)
        lv = q[:, 0] - 1
        b = self._bpa[lv]
        idx = self._off[lv] + (q[:, 1] * b + q[:, 2]) * b + q[:, 3]
        return [self._addrs[t] for t in idx.tolist()]


def _native(manifest) -> NativeManifest:
    nm = getattr(manifest, "_afam_native", None)
    if nm is None:
        nm = NativeManifest(manifest)
        try:
            object.__setattr__(manifest, "_afam_native", nm)
        except Exception:
            pass
    return nm


def select_visible(pov, manifest, aspect: float = 1.0, near: float = 1e-3, ranges=None) -> list:
    """Distance-banded LOD refinement + frustum culling (render.py:281-320), native."""
    return _native(manifest).select(pov, aspect, near, ranges)


# ------------------------------------------------------------- rendering
def camera_setup(pov, params) -> dict:
    f, r, u = pov_basis(pov)
    tan_y = math.tan(math.radians(pov.fov_y) / 2.0)
    return {"f": f, "r": r, "u": u, "tan_y": tan_y, "tan_x": tan_y * params.aspect}


def _frame_struct(pov, tf, params, band_rows, nparts, part, debug, full_frame=False) -> _lib.AfamFrame:
    # the TF and shading fields change rarely: a per-thread template keyed by
    # their values is copied and only the camera / band fields are set
    cp, op = np.asarray(tf.color_points, np.float64), np.asarray(tf.opacity_points, np.float64)
    key = (cp.tobytes(), op.tobytes(), cp.shape, op.shape, tuple(float(v) for v in tf.domain),
           float(params.sample_distance), params.reference_step, float(params.o_max), float(params.near),
           float(params.ambient), float(params.diffuse), float(params.specular), float(params.shininess))
    cache = getattr(_tls, "frame_tmpl", None)
    if cache is None or cache[0] != key:
        # TFs with more control points than the struct holds inline pass them
        # by pointer (afam_frame.color_pts / opacity_pts); the arrays live in
        # this cache entry, and libafam reads them only inside afam_render
        cpc, opc = np.ascontiguousarray(cp), np.ascontiguousarray(op)
        cache = (key, _frame_struct_full(pov, tf, params, band_rows, nparts, part, debug, full_frame), cpc, opc)
        _tls.frame_tmpl = cache
    fr = _lib.AfamFrame.from_buffer_copy(cache[1])
    if cache[2].shape[0] > _lib.AFAM_MAX_TF_POINTS or cache[3].shape[0] > _lib.AFAM_MAX_TF_POINTS:
        fr.color_pts, fr.opacity_pts = cache[2].ctypes.data, cache[3].ctypes.data
    cam = camera_setup(pov, params)
    for a in range(3):
        fr.origin[a] = float(pov.position[a])
        fr.f[a], fr.r[a], fr.u[a] = float(cam["f"][a]), float(cam["r"][a]), float(cam["u"][a])
    fr.tan_x, fr.tan_y = cam["tan_x"], cam["tan_y"]
    fr.width, fr.height = int(params.width), int(params.height)
    fr.band_rows, fr.nparts, fr.part = int(band_rows), int(nparts), int(part)
    fr.flags = (_lib.AFAM_RENDER_DEBUG if debug else 0) | (_lib.AFAM_RENDER_FULL_FRAME if full_frame else 0)
    return fr


def _frame_struct_full(pov, tf, params, band_rows, nparts, part, debug, full_frame=False) -> _lib.AfamFrame:
    fr = _lib.AfamFrame()
    cam = camera_setup(pov, params)
    for a in range(3):
        fr.origin[a] = float(pov.position[a])
        fr.f[a], fr.r[a], fr.u[a] = float(cam["f"][a]), float(cam["r"][a]), float(cam["u"][a])
    fr.tan_x, fr.tan_y = cam["tan_x"], cam["tan_y"]
    fr.width, fr.height = int(params.width), int(params.height)
    fr.band_rows, fr.nparts, fr.part = int(band_rows), int(nparts), int(part)
    sd = float(params.sample_distance)
    ref = params.reference_step if params.reference_step is not None else sd
    fr.sample_distance, fr.power, fr.o_max, fr.near_ = sd, sd / ref, float(params.o_max), float(params.near)
    fr.ambient, fr.diffuse = float(params.ambient), float(params.diffuse)
    fr.specular, fr.shininess = float(params.specular), float(params.shininess)
    cp, op = np.asarray(tf.color_points, np.float64), np.asarray(tf.opacity_points, np.float64)
    fr.ncolor, fr.nopacity = cp.shape[0], op.shape[0]
    for k in range(min(cp.shape[0], _lib.AFAM_MAX_TF_POINTS)):
        for c in range(4):
            fr.color[k][c] = float(cp[k, c])
    for k in range(min(op.shape[0], _lib.AFAM_MAX_TF_POINTS)):
        fr.opacity[k][0], fr.opacity[k][1] = float(op[k, 0]), float(op[k, 1])
    fr.domain_lo, fr.domain_hi = float(tf.domain[0]), float(tf.domain[1])
    fr.flags = (_lib.AFAM_RENDER_DEBUG if debug else 0) | (_lib.AFAM_RENDER_FULL_FRAME if full_frame else 0)
    return fr


def _missing_message(pov, params, cells, key) -> str:
    """Recompute the first uncovered sample exactly as render.py:422-436 would."""
    step, ray = key >> 32, key & 0xFFFFFFFF
    W, H = int(params.width), int(params.height)
    i, j = divmod(ray, W)
    cam = camera_setup(pov, params)
    xs = (j / W) * 2.0 - 1.0
    ys = 1.0 - (i / H) * 2.0
    px, py = xs * cam["tan_x"], ys * cam["tan_y"]
    d = [(cam["f"][a] + px * cam["r"][a]) + py * cam["u"][a] for a in range(3)]
    n = math.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
    d = [x / n for x in d]
    o = [float(v) for v in pov.position]
    te = -math.inf
    for a in range(3):
        inv = 1.0 / d[a] if d[a] != 0.0 else math.copysign(math.inf, d[a])
        ta, tb = (-1.0 - o[a]) * inv, (1.0 - o[a]) * inv
        lo = float(np.fmin(ta, tb))
        te = max(te, -math.inf if math.isnan(lo) else lo)
    te = max(te, float(params.near))
    t = te + (step + 0.5) * float(params.sample_distance)
    pos = [float(min(max(o[a] + t * d[a], -1.0), 1.0)) for a in range(3)]
    cell = tuple(min(max(int(((p + 1.0) / 2.0) * cells), 0), cells - 1) for p in pos)
    return (f"no resident block covers sample {pos} (finest cell {cell}); "
            "the resident set does not cover the visible region")


_tls = threading.local()


# A thread may have FRAMES_IN_FLIGHT submitted, uncollected frames (libafam
# keeps the same ring per thread, afam_render_seq): each ring entry has its
# own pinned staging buffer, device stats buffer and completion event.
FRAMES_IN_FLIGHT = 2


def _pinned_stage(nbytes: int, ring: int = 0):
    """This thread's pinned host staging buffer `ring` of >= 64 + nbytes bytes (grown on demand)."""
    import torch

    need = 64 + nbytes
    stages = getattr(_tls, "stages", None)
    if stages is None:
        stages = _tls.stages = [None] * FRAMES_IN_FLIGHT
    buf = stages[ring]
    if buf is None or buf.numel() < need:
        buf = torch.empty(max(need, 1 << 16), dtype=torch.uint8, pin_memory=True)
        stages[ring] = buf
    return buf


_streams: dict = {}


def _render_stream(dev):
    """A high-priority stream per (device, thread) for the render kernel:
    block uploads of the prefetch thread (default-priority loader streams)
    then yield the SMs to the frame.  render_part synchronizes it before
    returning, so callers see finished results as with their own stream."""
    import torch

    key = (dev.index, threading.get_ident())
    s = _streams.get(key)
    if s is None:
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        s = torch.cuda.Stream(device=dev, priority=min(lo, hi))
        _streams[key] = s
    return s


def render_part(pov, blocks: dict, tf, params, *, band_rows: int | None = None, nparts: int = 1, part: int = 0,
                device: int | None = None, debug: bool = False, stream=None, out=None, raise_missing=True,
                host_out: bool = False, out_ptr: int | None = None):
    """Render this part's row bands on the GPU.  Returns (rgba tensor (rows,
    W, 4) uint8 -- on the device, or in pinned host memory with host_out --,
    stats host dict, debug tensors or None).  Rows are the bands b with
    b % nparts == part, packed in band order.  With out_ptr (a device
    address of a whole H x W x 4 frame, e.g. rank 0's frame mapped over
    NVLink, tiles.PeerFrame) the rows land at their frame rows instead and
    the returned tensor is None."""
    return submit_part(pov, blocks, tf, params, band_rows=band_rows, nparts=nparts, part=part, device=device,
                       debug=debug, stream=stream, out=out, raise_missing=raise_missing, host_out=host_out,
                       out_ptr=out_ptr).result()


def _thread_stats(dev, ring: int = 0):
    """This thread's device stats buffer and completion event of ring entry `ring`."""
    import torch

    key = ("stats", dev.index)
    st = getattr(_tls, "stats", None)
    if st is None or st[0] != key:
        st = (key, [(torch.empty(7, dtype=torch.int64, device=dev), torch.cuda.Event())
                    for _ in range(FRAMES_IN_FLIGHT)])
        _tls.stats = st
    return st[1][ring]


def _addr_key(a):
    return (a.lod, a.ijk)


_inflight: dict = {}  # thread ident -> its uncollected PendingParts, oldest first (<= FRAMES_IN_FLIGHT)


class PendingPart:
    """A launched render_part: `done()` polls the GPU (no host wait),
    `result()` waits and returns render_part's (rgba, info, debug).  A thread
    has at most FRAMES_IN_FLIGHT uncollected frames (ring entries of staging
    buffer, stats buffer and completion event); a further submit waits for
    the oldest, whose result() then raises."""

    def __init__(self, **kw):
        self.__dict__.update(kw)
        self._res = None
        self._owner = threading.get_ident()
        _inflight.setdefault(self._owner, []).append(self)

    def done(self) -> bool:
        return self._res is not None or self.event.query()

    def result(self):
        if self._res is not None:
            return self._res
        import torch

        if getattr(self, "_superseded", False):
            raise RuntimeError("this frame's buffers were reused by a later submit on the same thread")
        mine = _inflight.get(self._owner)
        if mine is not None and self in mine:
            mine.remove(self)

        with torch.cuda.device(self.dev):
            self.event.synchronize()  # this frame only (a later frame may be queued behind it)
            st = self.stage[:56].view(torch.int64).numpy().copy()
            out = self.out
            if self.host_out:
                out = self.stage[64:64 + self.nbytes].view(self.rows, self.W, 4).clone()
        kms = C.c_float()
        _lib.check(_lib.lib().afam_render_elapsed_seq(self.store.handle, self.seq, C.byref(kms)))
        info = {"samples": int(st[0]), "missing_key": int(st[1]), "fp64_samples": int(st[2]),
                "shaded_samples": int(st[3]), "exact_samples": int(st[4]),
                "exact_cells": int(st[5]), "clear_samples": int(st[6]),
                "kernel_ms": float(kms.value)}
        if self.raise_missing and info["missing_key"] >= 0:
            cells = C.c_int32()
            _lib.check(_lib.lib().afam_owner_grid(self.store.handle, self.sl.ctypes.data_as(C.c_void_p),
                                                  len(self.sl), C.byref(cells), None, 0))
            raise MissingBlockError(_missing_message(self.pov, self.params, cells.value, info["missing_key"]))
        dbg = {"nsamp": self.nsamp, "ohash": self.ohash} if self.debug else None
        self._res = (out, info, dbg)
        return self._res


def submit_part(pov, blocks: dict, tf, params, *, band_rows: int | None = None, nparts: int = 1, part: int = 0,
                device: int | None = None, debug: bool = False, stream=None, out=None, raise_missing=True,
                host_out: bool = False, out_ptr: int | None = None) -> PendingPart:
    """render_part without the wait: launches the frame's kernels and
    returns a PendingPart, so the caller's thread can do host work (the
    replay prefetch) while the GPU marches."""
    import torch

    from .device import as_device_blocks, stream_handle

    ring = getattr(_tls, "nsubmit", 0) % FRAMES_IN_FLIGHT
    _tls.nsubmit = getattr(_tls, "nsubmit", 0) + 1
    mine = _inflight.setdefault(threading.get_ident(), [])
    for prev in [p for p in mine if p.ring == ring]:  # uncollected frame FRAMES_IN_FLIGHT submits ago:
        mine.remove(prev)                               # let it finish, its ring entry is reused
        prev.s_obj.synchronize()
        prev._superseded = True
    try:  # (lod, i, j, k) order as BlockAddress.__lt__, without a Python compare per pair
        addrs = sorted(blocks, key=_addr_key)
    except AttributeError:
        addrs = sorted(blocks)
    dev_index = torch.cuda.current_device() if device is None else int(device)
    store, slots = as_device_blocks([blocks[a] for a in addrs], dev_index)
    dev = torch.device("cuda", store.device)
    H, W = int(params.height), int(params.width)
    br = H if band_rows is None else int(band_rows)
    rows = int(_lib.lib().afam_frame_rows(H, br, nparts, part))
    fr = _frame_struct(pov, tf, params, br, nparts, part, debug, full_frame=out_ptr is not None)
    # host_out: the kernel stores the pixels straight into this thread's
    # pinned staging buffer (mapped host memory), overlapping the copy-out
    # with the march; one synchronization covers frame and stats
    if out_ptr is not None and host_out:
        raise ValueError("out_ptr and host_out are exclusive")
    zero_copy = host_out and out is None
    stage = _pinned_stage(rows * W * 4 if host_out else 0, ring)
    if out is None and out_ptr is None:
        out = stage[64:64 + rows * W * 4].view(rows, W, 4) if zero_copy else \
            torch.empty((rows, W, 4), dtype=torch.uint8, device=dev)
    stats, event = _thread_stats(dev, ring)
    nsamp = ohash = None
    if debug:
        nsamp = torch.empty((rows, W), dtype=torch.int32, device=dev)
        ohash = torch.empty((rows, W), dtype=torch.int64, device=dev)
    sl = np.ascontiguousarray(slots, dtype=np.int32)
    seq = C.c_uint64()
    with torch.cuda.device(dev):
        s_obj = stream if stream is not None else _render_stream(dev)
        _lib.check(_lib.lib().afam_render_seq(store.handle, C.byref(seq)))  # this call's number (kernel time)
        _lib.check(_lib.lib().afam_render(
            store.handle, C.byref(fr), sl.ctypes.data_as(C.c_void_p), len(sl),
            C.c_void_p(out_ptr if out_ptr is not None else out.data_ptr()),
            C.c_void_p(stats.data_ptr()), None if nsamp is None else C.c_void_p(nsamp.data_ptr()),
            None if ohash is None else C.c_void_p(ohash.data_ptr()), C.c_void_p(int(s_obj.cuda_stream))))
        with torch.cuda.stream(s_obj):
            stage[:56].view(torch.int64).copy_(stats, non_blocking=True)
            if host_out and not zero_copy:
                stage[64:64 + rows * W * 4].view(rows, W, 4).copy_(out, non_blocking=True)
            event.record(s_obj)
    return PendingPart(dev=dev, s_obj=s_obj, stage=stage, out=out, host_out=host_out, nbytes=rows * W * 4,
                       rows=rows, W=W, store=store, sl=sl, pov=pov, params=params, raise_missing=raise_missing,
                       debug=debug, nsamp=nsamp, ohash=ohash, stats=stats, event=event, seq=int(seq.value), ring=ring)


class PendingFrame:
    """render.submit's handle: `done()` polls, `result()` returns the Frame
    (and sets `on.last_stats`)."""

    def __init__(self, part: PendingPart, params, on, finish=None):
        self.part, self.params, self.on, self.finish = part, params, on, finish

    def done(self) -> bool:
        return self.part.done()

    def result(self):
        out, info, _ = self.part.result()
        self.on.last_stats = info
        if self.finish is not None:
            return self.finish(out, info)
        return Frame(width=int(self.params.width), height=int(self.params.height), rgba=out.numpy())


def submit(pov, blocks: dict, tf, params) -> PendingFrame:
    """render() split at the GPU wait: launch the frame, return a handle."""
    return PendingFrame(submit_part(pov, blocks, tf, params, host_out=True), params, render)


def render(pov, blocks: dict, tf, params) -> Frame:
    """Front-to-back composite of the resident blocks (render.py:398-466) on the GPU."""
    return submit(pov, blocks, tf, params).result()


render.submit = submit
render.last_stats = None
render.frames_in_flight = FRAMES_IN_FLIGHT  # runtime.replay may launch frame i+1 before collecting frame i
