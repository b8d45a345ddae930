"""Adaptive per-block NCP search and cross-level encoding on the GPU.

Same API and decisions as the reference encoder (encoder.py:1-285): every
searched block gets the smallest control-point count (NCP) whose
reconstruction RMSE beats the error bound -- a full sweep from the block edge
down to degree+1, or a bisection with assume_monotone -- a block is complex
when it needs more than the minimum, and the adaptive mode searches a finer
block only when its parent was complex.

The inner loop (reference _fit_and_measure: model.fit + error_rmse,
encoder.py:74-83) runs in libafam (afam_fit_rmse): for a batch of (block,
NCP) jobs the endpoint-pinned separable least-squares fit, the float32
rounding of the coefficients, the dense decode onto the sample lattice and
the RMSE, all float64 like the reference.  The host drives the search: a
full sweep is one batch per level (every block x every NCP), a bisection
advances all blocks of a level in lockstep, one batch per probe round.
"""

from __future__ import annotations

import ctypes as C
import threading
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib, model
from .partition import BlockAddress, build_hierarchy

__all__ = ["ErrorProfile", "SearchResult", "EncodeStats", "error_rmse", "fit_rmse_batch", "search_blocks",
           "in_level_search", "cross_level_encode", "compression_ratio", "encode_volume"]


@dataclass
class ErrorProfile:
    """NCP -> reconstruction RMSE for one block (dense for a full sweep)."""

    rmse_by_ncp: dict = field(default_factory=dict)

    def record(self, ncp: int, rmse: float) -> None:
        self.rmse_by_ncp[int(ncp)] = float(rmse)


@dataclass
class SearchResult:
    ncp_star: int
    profile: ErrorProfile
    is_complex: bool
    met_bound: bool
    model: model.MicroModel


@dataclass
class EncodeStats:
    total_blocks: int = 0
    searched_blocks: int = 0
    searched_by_level: dict = field(default_factory=dict)
    complex_by_level: dict = field(default_factory=dict)
    unmet_blocks: list = field(default_factory=list)

    def to_json(self) -> dict:
        return {"total_blocks": self.total_blocks, "searched_blocks": self.searched_blocks,
                "searched_by_level": {str(k): v for k, v in sorted(self.searched_by_level.items())},
                "complex_by_level": {str(k): v for k, v in sorted(self.complex_by_level.items())},
                "unmet_blocks": list(self.unmet_blocks)}


_stores: dict = {}
_stores_lock = threading.Lock()
WORK_BYTES = 4 << 30  # device scratch per batch: 2 float64 m^3 buffers per job


def _op_store(device: int):
    """A 1-slot DeviceStore per device: afam_fit_rmse's device and operator cache."""
    from .device import DeviceStore

    with _stores_lock:
        if device not in _stores:
            _stores[device] = DeviceStore(1, 9, device)
        return _stores[device]


def fit_rmse_batch(samples, degree: int, jobs, want_ctrl: bool = False, device: int = 0):
    """Run (block index, ncp) jobs over a list of float32 sample grids of one
    shape (d0, d1, d2) (bspline.fit_tensor_product fits any 3-D grid; cubic
    in the configs).  Returns rmse (njobs,) and, with want_ctrl, the list of
    float32 (ncp, ncp, ncp) coefficient grids (C order, [a, b, c] = x, y, z)."""
    import torch

    _lib.require_device()
    dev = torch.device("cuda", device)
    if isinstance(samples, torch.Tensor):  # already resident: (nblk, d0, d1, d2) float32 on `device`
        d_samples = samples.contiguous()
        nblk, dims = int(d_samples.shape[0]), tuple(int(v) for v in d_samples.shape[1:])
    else:
        blocks = [np.ascontiguousarray(s, dtype=np.float32) for s in samples]
        if not blocks:
            return np.zeros(0), ([] if want_ctrl else None)
        dims = tuple(blocks[0].shape)
        if len(dims) != 3:
            raise ValueError("expected a 3D sample grid")
        if any(b.shape != dims for b in blocks):
            raise ValueError("fit_rmse_batch needs sample grids of one shape")
        nblk = len(blocks)
        d_samples = torch.from_numpy(np.stack(blocks)).to(dev)
    jobs = [(int(b), int(n)) for b, n in jobs]
    for _, n in jobs:  # bspline.fit_tensor_product's check, axis by axis
        for axis, d in enumerate(dims):
            if not degree + 1 <= n <= d:
                raise ValueError(f"ncp must be in [{degree + 1}, {d}] for axis {axis}, got {n}")
    c_dims = (C.c_int32 * 3)(*dims)
    store = _op_store(device)
    per = max(1, min(65535, WORK_BYTES // (16 * int(np.prod(dims)))))
    rmse = np.zeros(len(jobs))
    ctrls = [] if want_ctrl else None
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        for s0 in range(0, len(jobs), per):
            chunk = jobs[s0:s0 + per]
            jb = np.array([b for b, _ in chunk], dtype=np.int32)
            jn = np.array([n for _, n in chunk], dtype=np.int32)
            out = np.zeros(len(chunk))
            d_ctrl, offs = None, None
            if want_ctrl:
                sizes = jn.astype(np.int64) ** 3
                offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
                d_ctrl = torch.empty(int(sizes.sum()), dtype=torch.float32, device=dev)
            _lib.check(_lib.lib().afam_fit_rmse3(
                store.handle, C.c_void_p(d_samples.data_ptr()), nblk, c_dims, int(degree),
                jb.ctypes.data_as(C.c_void_p), jn.ctypes.data_as(C.c_void_p), len(chunk),
                out.ctypes.data_as(C.c_void_p), None if d_ctrl is None else C.c_void_p(d_ctrl.data_ptr()),
                None if offs is None else offs.ctypes.data_as(C.c_void_p), C.c_void_p(stream.cuda_stream)))
            rmse[s0:s0 + len(chunk)] = out
            if want_ctrl:
                host = d_ctrl.cpu().numpy()
                for n, o in zip(jn, offs):
                    ctrls.append(host[o:o + int(n) ** 3].reshape(int(n), int(n), int(n)).copy())
    return rmse, ctrls


def _make_model(ctrl, degree, extent, lod) -> model.MicroModel:
    from .bspline import clamped_knots

    knots = clamped_knots(ctrl.shape[0], degree).astype(np.float32)
    return model.MicroModel(degree, np.repeat(knots[None, :], 3, axis=0), ctrl.astype(np.float32),
                            np.asarray(extent, dtype=np.float64), lod)


def search_blocks(samples, error_bound: float, degree: int, extents=None, lods=None,
                  assume_monotone: bool = False, device: int = 0) -> list:
    """in_level_search for many blocks of one shape at once (one GPU batch per
    sweep / bisection round).  `samples`: a list of host arrays or a
    resident (nblocks, d0, d1, d2) float32 CUDA tensor; NCPs run up to the
    edge d0 as the reference's (encoder.py:104).  Returns [SearchResult]."""
    import torch

    if error_bound <= 0:
        raise ValueError("error bound must be positive")
    on_device = isinstance(samples, torch.Tensor)
    blocks = samples if on_device else [np.asarray(s) for s in samples]
    nb = len(blocks)
    if nb == 0:
        return []
    n = int(blocks[0].shape[0])
    ncp_min = degree + 1
    if n < ncp_min:
        raise ValueError(f"block edge {n} below minimum NCP {ncp_min}")
    extents = extents if extents is not None else [((0.0, 1.0),) * 3] * nb
    lods = lods if lods is not None else [1] * nb
    profiles = [ErrorProfile() for _ in range(nb)]
    _lib.require_device()
    shape = tuple(int(v) for v in blocks[0].shape)
    if on_device:  # (nb, d0, d1, d2) float32, already resident
        if blocks.dim() != 4 or blocks.dtype != torch.float32:
            raise ValueError("search_blocks needs a (nblocks, d0, d1, d2) float32 tensor")
        blocks = blocks.contiguous()
    else:
        if any(np.shape(b) != shape for b in blocks):
            raise ValueError("search_blocks needs sample grids of one shape")
        blocks = torch.from_numpy(np.stack([np.asarray(b, dtype=np.float32) for b in blocks])).to(
            torch.device("cuda", device))  # uploaded once for every probe round
    if assume_monotone:
        lo, hi = [ncp_min] * nb, [n] * nb
        while True:
            active = [b for b in range(nb) if lo[b] < hi[b]]
            if not active:
                break
            mids = {b: (lo[b] + hi[b]) // 2 for b in active}
            r, _ = fit_rmse_batch(blocks, degree, [(b, mids[b]) for b in active], device=device)
            for b, v in zip(active, r):
                profiles[b].record(mids[b], v)
                if v < error_bound:
                    hi[b] = mids[b]
                else:
                    lo[b] = mids[b] + 1
        todo = [b for b in range(nb) if lo[b] not in profiles[b].rmse_by_ncp]
        if todo:
            r, _ = fit_rmse_batch(blocks, degree, [(b, lo[b]) for b in todo], device=device)
            for b, v in zip(todo, r):
                profiles[b].record(lo[b], v)
        met = [profiles[b].rmse_by_ncp[lo[b]] < error_bound for b in range(nb)]
        star = [lo[b] if met[b] else n for b in range(nb)]
    else:
        jobs = [(b, ncp) for b in range(nb) for ncp in range(n, ncp_min - 1, -1)]
        r, _ = fit_rmse_batch(blocks, degree, jobs, device=device)
        for (b, ncp), v in zip(jobs, r):
            profiles[b].record(ncp, v)
        star, met = [], []
        for b in range(nb):
            good = [ncp for ncp, v in profiles[b].rmse_by_ncp.items() if v < error_bound]
            met.append(bool(good))
            star.append(min(good) if good else n)
    for b in range(nb):
        if not met[b]:
            warnings.warn(f"error bound {error_bound:g} unmeetable for block "
                          f"(best rmse {min(profiles[b].rmse_by_ncp.values()):.3g}); using ncp={n}",
                          RuntimeWarning, stacklevel=2)
    # the chosen models: one more (cheap) batch that also returns the coefficients
    need = [(b, star[b]) for b in range(nb)]
    r, ctrls = fit_rmse_batch(blocks, degree, need, want_ctrl=True, device=device)
    out = []
    for b in range(nb):
        if star[b] not in profiles[b].rmse_by_ncp:  # bisection landing on n without having fit it
            profiles[b].record(star[b], r[b])
        out.append(SearchResult(ncp_star=star[b], profile=profiles[b], is_complex=star[b] > ncp_min,
                                met_bound=met[b], model=_make_model(ctrls[b], degree, extents[b], lods[b])))
    return out


def in_level_search(samples, error_bound: float, degree: int, extent=((0.0, 1.0),) * 3, lod: int = 1,
                    assume_monotone: bool = False) -> SearchResult:
    """Smallest NCP whose RMSE beats the bound for one block (reference
    encoder.py:86-156)."""
    return search_blocks([samples], error_bound, degree, [extent], [lod], assume_monotone)[0]


def error_rmse(samples, block_model) -> float:
    """RMSE between the model decoded on the sample lattice and the samples
    (reference encoder.py:74-78; decode on the GPU, K3)."""
    decoded = block_model.decode_grid(np.asarray(samples).shape)
    diff = decoded - np.asarray(samples, dtype=np.float64)
    return float(np.sqrt(np.mean(diff * diff)))


def _fixed(samples_list, ncp_list, degree, extents, lods):
    """Fit at given NCPs (the reference's _encode_fixed)."""
    if not samples_list:
        return []
    _, ctrls = fit_rmse_batch(samples_list, degree, [(b, n) for b, n in enumerate(ncp_list)], want_ctrl=True)
    return [_make_model(c, degree, e, l) for c, e, l in zip(ctrls, extents, lods)]


def cross_level_encode(manifest, blocks: dict, error_bound: float, degree: int = 2, mode: str = "adaptive",
                       assume_monotone: bool = False, workers: int | None = None):
    """Encode every block, coarsest level first (reference encoder.py:166-255):
    "adaptive" searches a block only when its parent was complex, "exhaustive"
    searches every block, "fixed:<ncp>" fits everything at one NCP.  Fills the
    manifest's ncp/is_complex/nbytes in place; returns (models, stats).
    `workers` is accepted for API compatibility (the GPU batches a level)."""
    if mode not in ("adaptive", "exhaustive") and not mode.startswith("fixed:"):
        raise ValueError(f"unknown encode mode {mode!r}")
    stats = EncodeStats(total_blocks=len(blocks))
    models, complex_at = {}, set()
    ncp_min = degree + 1
    manifest.degree = degree
    manifest.error_bound = error_bound
    for lod in range(manifest.levels, 0, -1):
        addrs = manifest.addresses(lod)
        if mode == "adaptive":
            searched = [a for a in addrs if lod == manifest.levels or a.parent() in complex_at]
        elif mode == "exhaustive":
            searched = list(addrs)
        else:
            searched = []
        results = {}
        if searched:
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                res = search_blocks([blocks[a].samples for a in searched], error_bound, degree,
                                    [manifest.entries[a].extent for a in searched], [a.lod for a in searched],
                                    assume_monotone)
            results = dict(zip(searched, res))
            for w in caught:
                warnings.warn(str(w.message), RuntimeWarning, stacklevel=2)
        fixed_ncp = int(mode.split(":", 1)[1]) if mode.startswith("fixed:") else ncp_min
        skipped = [a for a in addrs if a not in results]
        fixed_ncps = [min(max(fixed_ncp, ncp_min), blocks[a].samples.shape[0]) for a in skipped]
        fixed_models = dict(zip(skipped, _fixed([blocks[a].samples for a in skipped], fixed_ncps, degree,
                                                [manifest.entries[a].extent for a in skipped],
                                                [a.lod for a in skipped])))
        for addr in addrs:  # deterministic manifest fill order
            entry = manifest.entries[addr]
            if addr in results:
                r = results[addr]
                models[addr] = r.model
                entry.ncp, entry.is_complex = r.ncp_star, r.is_complex
                if not r.met_bound:
                    stats.unmet_blocks.append(addr.key)
                if r.is_complex:
                    complex_at.add(addr)
                stats.searched_blocks += 1
                stats.searched_by_level[lod] = stats.searched_by_level.get(lod, 0) + 1
            else:
                models[addr] = fixed_models[addr]
                entry.ncp = models[addr].control.shape[0]
                entry.is_complex = False
            entry.nbytes = model.serialized_size(entry.ncp, degree)
        stats.complex_by_level[lod] = sum(1 for a in addrs if manifest.entries[a].is_complex)
    return models, stats


def compression_ratio(manifest, raw_bytes: int) -> float:
    """Raw volume bytes over the byte total of every model, all levels."""
    return raw_bytes / manifest.total_model_bytes()


def encode_volume(vol, levels: int, micro_dims, degree: int = 2, error_bound: float = 1e-4, coarsest: int = 2,
                  mode: str = "adaptive", assume_monotone: bool = False, workers: int | None = None):
    """Partition + encode in one call; returns (manifest, models, stats)
    (reference encoder.py:258-285).  `vol` has .samples (3-D) and .bounds (3, 2)."""
    manifest, blocks = build_hierarchy(vol, levels, micro_dims, coarsest=coarsest)
    models, stats = cross_level_encode(manifest, blocks, error_bound, degree=degree, mode=mode,
                                       assume_monotone=assume_monotone, workers=workers)
    return manifest, models, stats
