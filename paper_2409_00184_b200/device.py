"""HBM-resident micro-model store (host side of the K4 upload path).

A DeviceStore owns `slots` fixed-size slots on one GPU (libafam
afam_store_*).  Models enter a slot either as raw .mfa file images
(put_mfa: the misaligned file bytes go H2D verbatim and are realigned on
device) or as decoded arrays (put_model).  DeviceBlock is the handle the
loader/cache hand to render(); it satisfies the reference's block protocol
attributes (.extent, .lod, .nbytes; reference render.py:3-7,
runtime.py:132) plus .slot/.store.

Plain MicroModels passed to render()/decode_grid()/values_at() are
uploaded on demand into a per-process scratch store (an LRU keyed by the
model object), as SURVEY.md 8(b) prescribes for the CLI path.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib
from .errors import CapacityError, FormatError

__all__ = ["DeviceStore", "DeviceBlock", "scratch_store", "stream_handle", "as_device_blocks"]


def serialized_size(ncp: int, degree: int) -> int:
    return 1 + ((ncp + degree) * 3 + ncp ** 3) * 4


def check_mfa(data, ncp: int) -> int:
    """Validate a host .mfa image like afam_store_put_mfa (FormatError /
    ValueError); returns its degree byte."""
    buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    deg = C.c_int32(0)
    _lib.check(_lib.lib().afam_mfa_check(buf.ctypes.data_as(C.c_void_p), buf.size, int(ncp), C.byref(deg)))
    return int(deg.value)


def stream_handle(stream=None, device=None) -> int:
    """cudaStream_t (as int) of a torch stream, or torch's current stream."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream)


class DeviceBlock:
    """Handle to a model resident in a DeviceStore slot."""

    __slots__ = ("store", "slot", "extent", "lod", "degree", "ncp", "nbytes", "kind", "__weakref__")

    def __init__(self, store, slot, extent, lod, degree, ncp, kind: str = "mfa", nbytes: int | None = None):
        self.store = store
        self.slot = int(slot)
        self.extent = np.asarray(extent, dtype=np.float64).reshape(3, 2)
        self.lod = int(lod)
        self.degree = int(degree)  # DS blocks: the ghost width
        self.ncp = int(ncp)        # DS blocks: the largest interior lattice dim
        self.kind = kind
        self.nbytes = int(nbytes) if nbytes is not None else serialized_size(self.ncp, self.degree)

    def values_at(self, points):
        from .bspline import eval_device

        return eval_device(self.store, self.slot, points, gradient=False)

    def gradients_at(self, points):
        from .bspline import eval_device

        return eval_device(self.store, self.slot, points, gradient=True)[1]

    def decode_grid(self, dims):
        from .bspline import decode_block

        return decode_block(self.store, self.slot, dims)

    def __repr__(self):
        return f"DeviceBlock(slot={self.slot}, lod={self.lod}, ncp={self.ncp}, degree={self.degree})"


def _extent6(extent) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(extent, dtype=np.float64).reshape(3, 2).ravel())


class DeviceStore:
    """`slots` micro-model slots of up to `max_ncp` control points per axis."""

    def __init__(self, slots: int, max_ncp: int, device: int = 0, fp64_ctrl_limit: float = 4.0):
        _lib.require_device()
        self.device = int(device)
        self.slots = int(slots)
        self.max_ncp = int(max_ncp)
        h = C.c_void_p()
        _lib.check(_lib.lib().afam_store_create(C.byref(h), self.device, self.slots, self.max_ncp,
                                                float(fp64_ctrl_limit)))
        self._h = h
        self._free = list(range(self.slots - 1, -1, -1))
        self._lock = threading.Lock()
        self._fin = weakref.finalize(self, _lib.lib().afam_store_destroy, h)

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------- slots
    def alloc(self) -> int:
        with self._lock:
            if not self._free:
                raise CapacityError(f"all {self.slots} device slots are in use")
            return self._free.pop()

    def release(self, slot: int) -> None:
        _lib.check(_lib.lib().afam_store_evict(self._h, int(slot)))
        with self._lock:
            self._free.append(int(slot))

    def free_slots(self) -> int:
        with self._lock:
            return len(self._free)

    # ------------------------------------------------------------- uploads
    def put_mfa(self, slot: int, data, ncp: int, extent, stream=None) -> None:
        """Upload one .mfa file image (FORMAT.md:16-70).  Length / degree-byte
        violations raise FormatError like model.deserialize (model.py:121-133)."""
        buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        ext = _extent6(extent)
        _lib.check(_lib.lib().afam_store_put_mfa(self._h, int(slot), buf.ctypes.data_as(C.c_void_p), buf.size,
                                                 int(ncp), ext.ctypes.data_as(C.c_void_p),
                                                 C.c_void_p(stream_handle(stream, self.device))))

    def put_mfa_device(self, slot: int, dptr: int, nbytes: int, degree: int, ncp: int, extent, stream=None) -> None:
        """Upload a .mfa image that already sits in device memory (validated
        on the host by check_mfa): D2D copy + realignment."""
        ext = _extent6(extent)
        _lib.check(_lib.lib().afam_store_put_mfa_device(self._h, int(slot), C.c_void_p(int(dptr)), int(nbytes),
                                                        int(degree), int(ncp), ext.ctypes.data_as(C.c_void_p),
                                                        C.c_void_p(stream_handle(stream, self.device))))

    def put_file(self, slot: int, path, ncp: int, extent, stream=None) -> int:
        """Upload one .mfa file from disk through the native pinned staging
        ring (afam_store_put_file); returns the file's degree byte."""
        ext = _extent6(extent)
        deg = C.c_int32(0)
        _lib.check(_lib.lib().afam_store_put_file(self._h, int(slot), str(path).encode(), int(ncp),
                                                  ext.ctypes.data_as(C.c_void_p), C.byref(deg),
                                                  C.c_void_p(stream_handle(stream, self.device))))
        return int(deg.value)

    def load_file(self, path, ncp: int, extent, lod: int, stream=None) -> DeviceBlock:
        slot = self.alloc()
        try:
            deg = self.put_file(slot, path, ncp, extent, stream)
        except Exception:
            with self._lock:
                self._free.append(slot)
            raise
        return DeviceBlock(self, slot, extent, lod, deg, ncp)

    def put_ds(self, slot: int, data, extent, stream=None) -> None:
        """Upload one DS block file image (afam_store_put_ds)."""
        buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        _lib.check(_lib.lib().afam_store_put_ds(self._h, int(slot), buf.ctypes.data_as(C.c_void_p), buf.size,
                                                _extent6(extent).ctypes.data_as(C.c_void_p),
                                                C.c_void_p(stream_handle(stream, self.device))))

    def load_ds(self, data, extent, lod: int, stream=None) -> DeviceBlock:
        import struct

        slot = self.alloc()
        try:
            self.put_ds(slot, data, extent, stream)
        except Exception:
            with self._lock:
                self._free.append(slot)
            raise
        nx, ny, nz, g = struct.unpack_from("<4I", bytes(data[:16]))
        return DeviceBlock(self, slot, extent, lod, g, max(nx, ny, nz) - 2 * g, kind="ds", nbytes=len(data))

    def put_model(self, slot: int, model, stream=None) -> None:
        ctrl = np.ascontiguousarray(np.asarray(model.control, dtype=np.float32).ravel(order="F"))
        knots = np.ascontiguousarray(np.asarray(model.knots, dtype=np.float32))
        ncp = int(np.asarray(model.control).shape[0])
        ext = _extent6(model.extent)
        _lib.check(_lib.lib().afam_store_put(self._h, int(slot), int(model.degree), ncp,
                                             knots.ctypes.data_as(C.c_void_p), ctrl.ctypes.data_as(C.c_void_p),
                                             ext.ctypes.data_as(C.c_void_p),
                                             C.c_void_p(stream_handle(stream, self.device))))

    def load_mfa(self, data, ncp: int, extent, lod: int, stream=None) -> DeviceBlock:
        slot = self.alloc()
        try:
            self.put_mfa(slot, data, ncp, extent, stream)
        except Exception:
            with self._lock:
                self._free.append(slot)
            raise
        return DeviceBlock(self, slot, extent, lod, int(np.frombuffer(data, dtype=np.uint8, count=1)[0]), ncp)

    def load_model(self, model, stream=None) -> DeviceBlock:
        slot = self.alloc()
        try:
            self.put_model(slot, model, stream)
        except Exception:
            with self._lock:
                self._free.append(slot)
            raise
        return DeviceBlock(self, slot, model.extent, getattr(model, "lod", 1), model.degree,
                           np.asarray(model.control).shape[0])

    # ------------------------------------------------------------- queries
    def info(self, slot: int):
        ncp, deg, flags, mx = C.c_int32(), C.c_int32(), C.c_uint32(), C.c_float()
        _lib.check(_lib.lib().afam_store_info(self._h, int(slot), C.byref(ncp), C.byref(deg), C.byref(flags),
                                              C.byref(mx)))
        return {"ncp": ncp.value, "degree": deg.value, "fp64": bool(flags.value & _lib.AFAM_SLOT_FP64),
                "max_abs_ctrl": mx.value}

    def read(self, slot: int):
        inf = self.info(slot)
        n, d = inf["ncp"], inf["degree"]
        ctrl = np.zeros(n ** 3, dtype=np.float32)
        knots = np.zeros(3 * (n + d + 1), dtype=np.float32)
        _lib.check(_lib.lib().afam_store_read(self._h, int(slot), ctrl.ctypes.data_as(C.c_void_p),
                                              knots.ctypes.data_as(C.c_void_p)))
        return ctrl.reshape((n, n, n), order="F"), knots.reshape(3, n + d + 1)


# --------------------------------------------------------------- scratch
_BUCKETS = (9, 17, 33, 65, 129, 257)
_scratch: dict = {}
_scratch_lock = threading.Lock()


class _ScratchStore:
    """LRU of host models uploaded on demand into one DeviceStore."""

    def __init__(self, max_ncp: int, device: int):
        slot_bytes = 9 * 4 * max_ncp ** 3 + 65536  # raw + pitched + x-quad control points + cell ranges + tables
        slots = int(min(1024, max(16, (2 << 30) // slot_bytes)))
        self.store = DeviceStore(slots, max_ncp, device)
        self.lru: OrderedDict = OrderedDict()  # id(model) -> (weakref or None, DeviceBlock)
        self.lock = threading.Lock()

    def get(self, model, pinned=()) -> DeviceBlock:
        key = id(model)
        with self.lock:
            hit = self.lru.get(key)
            # objects that cannot be weakly referenced are never reused: id() may be recycled
            if hit is not None and hit[0] is not None and hit[0]() is model:
                self.lru.move_to_end(key)
                return hit[1]
            if hit is not None:
                self._drop(key)
            while self.store.free_slots() == 0:
                victim = next((k for k in self.lru if k not in pinned), None)
                if victim is None:
                    raise CapacityError("scratch device store is full of pinned blocks")
                self._drop(victim)
            blk = self.store.load_model(model)
            try:
                ref = weakref.ref(model)
            except TypeError:
                ref = None
            self.lru[key] = (ref, blk)
            return blk

    def get_ds(self, block, serialize, pinned=()) -> DeviceBlock:
        """Upload (or reuse) a host DS block, keyed like get(); blocks of the
        current call (`pinned` ids) are never evicted to make room."""
        key = id(block)
        with self.lock:
            hit = self.lru.get(key)
            if hit is not None and hit[0] is not None and hit[0]() is block:
                self.lru.move_to_end(key)
                return hit[1]
            if hit is not None:
                self._drop(key)
            while self.store.free_slots() == 0:
                victim = next((k for k in self.lru if k not in pinned), None)
                if victim is None:
                    raise CapacityError("scratch device store is full of pinned blocks")
                self._drop(victim)
            blk = self.store.load_ds(serialize(block), block.extent, block.lod)
            try:
                ref = weakref.ref(block)
            except TypeError:
                ref = None
            self.lru[key] = (ref, blk)
            return blk

    def _drop(self, key):
        _, blk = self.lru.pop(key)
        self.store.release(blk.slot)


def scratch_store(max_ncp: int, device: int = 0, exact: bool = False) -> _ScratchStore:
    """The per-process scratch store for host models of up to `max_ncp`
    control points per axis (size buckets); `exact` sizes the slots for
    exactly `max_ncp` (DS blocks: the ghosted sample edge)."""
    bucket = int(max_ncp) if exact else next((b for b in _BUCKETS if b >= max_ncp), None)
    if bucket is None:
        bucket = int(max_ncp)
    with _scratch_lock:
        key = (bucket, int(device), bool(exact))
        if key not in _scratch:
            _scratch[key] = _ScratchStore(bucket, device)
        return _scratch[key]


def as_device_blocks(values, device: int = 0):
    """Resolve a sequence of blocks (DeviceBlock or MicroModel-like) to
    (store, [slots]) in one DeviceStore, uploading host models as needed."""
    values = list(values)
    stores = {id(v.store): v.store for v in values if isinstance(v, DeviceBlock)}
    hosts = [v for v in values if not isinstance(v, DeviceBlock)]
    if not hosts and len(stores) == 1:
        return next(iter(stores.values())), [v.slot for v in values]
    if not hosts and not values:
        return scratch_store(9, device).store, []
    from .downsample import DsBlock, serialize_ds

    if hosts and all(isinstance(v, DsBlock) for v in hosts):  # DS baseline blocks
        edge = max(max(v.samples.shape) for v in hosts) if hosts else 9
        sc = scratch_store(edge, device, exact=True)  # DS slots sized by the sample edge, not a spline bucket
        pinned = set(id(v) for v in values)
        slots = []
        for v in values:
            if isinstance(v, DeviceBlock):
                raise TypeError("cannot mix resident DeviceBlocks with host DS blocks in one render")
            slots.append(sc.get_ds(v, serialize_ds, pinned).slot)
        return sc.store, slots
    for v in hosts:
        if not (hasattr(v, "control") and hasattr(v, "knots") and hasattr(v, "degree") and hasattr(v, "extent")):
            raise TypeError(f"block {type(v).__name__} is not a spline micro-model or DS block; the B200 path "
                            "decodes MicroModel/DsBlock/DeviceBlock blocks only (no CPU fallback)")
    max_ncp = max(int(v.ncp) if isinstance(v, DeviceBlock) else int(np.asarray(v.control).shape[0]) for v in values)
    sc = scratch_store(max_ncp, device)
    pinned = set(id(v) for v in values)
    slots = []
    for v in values:
        if isinstance(v, DeviceBlock) and v.store is sc.store:
            slots.append(v.slot)
            continue
        if isinstance(v, DeviceBlock):  # resident in another store: stage through the host
            ctrl, knots = v.store.read(v.slot)
            from types import SimpleNamespace

            v = SimpleNamespace(control=ctrl, knots=knots, degree=v.degree, extent=v.extent, lod=v.lod)
        slots.append(sc.get(v, pinned).slot)
    return sc.store, slots
