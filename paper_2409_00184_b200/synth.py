"""Synthetic Adaptive-FAM stores for benchmarks and GPU parity tests.

Input synthesis only (not on the decode/render path).  Blocks are fitted
with the endpoint-pinned least-squares operator the reference encoder uses
(reference bspline.py:109-159: end coefficients pinned to the end samples,
interior coefficients from the normal equations), restated here
independently so stores can be built on a GPU box without the reference.

`turbulence_store` is BASELINE config 3 (1024^3-equivalent: 1025^3
lattice, 4 LODs, coarsest 2, micro 65 -> 4,680 blocks): a seeded sum of K
Fourier modes with a k^(-5/3) amplitude spectrum, normalized to ~[0, 1].
Because the fit is linear and each mode is separable,
exp(i 2pi k.x) = prod_a exp(i 2pi k_a x_a), a block's control grid is
Re sum_K A_K (P e_x,K) (x) (P e_y,K) (x) (P e_z,K) -- no 65^3 sampling.
"""

from __future__ import annotations

import hashlib
from functools import lru_cache

import numpy as np

from .bspline import clamped_knots
from .partition import BlockAddress, ManifestEntry, block_extent, skeleton

__all__ = ["fit_operator", "turbulence_store", "ml_value", "ml_volume", "field_store", "ncp_for", "pack_mfa"]

SEED = 20261017


def _basis_rows(params: np.ndarray, knots: np.ndarray, ncp: int, degree: int) -> np.ndarray:
    """Dense (len(params), ncp) collocation matrix by Cox-de Boor."""
    n = params.shape[0]
    span = np.clip(np.searchsorted(knots, params, side="right") - 1, degree, ncp - 1)
    vals = np.zeros((n, degree + 1))
    vals[:, 0] = 1.0
    for j in range(1, degree + 1):
        prev = vals.copy()
        vals[:] = 0.0
        for r in range(j):
            lo_k = knots[span + r + 1 - j]
            hi_k = knots[span + r + 1]
            w = prev[:, r] / (hi_k - lo_k)
            vals[:, r] += (hi_k - params) * w
            vals[:, r + 1] += (params - lo_k) * w
    B = np.zeros((n, ncp))
    cols = span[:, None] - degree + np.arange(degree + 1)[None, :]
    B[np.arange(n)[:, None], cols] = vals
    return B


@lru_cache(maxsize=256)
def fit_operator(m: int, ncp: int, degree: int) -> np.ndarray:
    """(ncp, m) operator: uniform samples -> endpoint-pinned LSQ coefficients."""
    B = _basis_rows(np.linspace(0.0, 1.0, m), clamped_knots(ncp, degree), ncp, degree)
    P = np.zeros((ncp, m))
    P[0, 0] = 1.0
    P[-1, -1] = 1.0
    if ncp > 2:
        Bi = B[:, 1:-1]
        R = np.eye(m)
        R[:, 0] -= B[:, 0]
        R[:, -1] -= B[:, -1]
        P[1:-1] = np.linalg.solve(Bi.T @ Bi, Bi.T @ R)
    return P


def ncp_for(addr: BlockAddress, lo: int = 40, hi: int = 65) -> int:
    """Deterministic per-block control-point count in [lo, hi] (an adaptive
    encoder's spread of NCPs; the top two values are the ill-conditioned
    ncp >= m-1 regime of SURVEY.md sec. 7)."""
    h = int.from_bytes(hashlib.blake2b(addr.key.encode(), digest_size=4).digest(), "little")
    return hi - h % (hi - lo + 1)


def pack_mfa(degree: int, control: np.ndarray) -> bytes:
    """FORMAT.md:16-70 image of a clamped-uniform model."""
    ncp = control.shape[0]
    kv = clamped_knots(ncp, degree).astype("<f4")
    return bytes([degree]) + kv[1:].tobytes() * 3 + np.asarray(control, dtype="<f4").ravel(order="F").tobytes()


def _modes(K: int, seed: int, kmax: float):
    rng = np.random.default_rng(seed)
    dirs = rng.normal(size=(K, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    kmag = np.exp(rng.uniform(np.log(1.0), np.log(kmax), size=K))
    kvec = dirs * kmag[:, None]
    amp = kmag ** (-5.0 / 3.0)
    phase = rng.uniform(0, 2 * np.pi, size=K)
    return kvec, amp * np.exp(1j * phase)


def _mode_factors(P: np.ndarray, lo: float, hi: float, m: int, k: np.ndarray) -> np.ndarray:
    xs = lo + (hi - lo) * (np.arange(m) / (m - 1))
    return P @ np.exp(2j * np.pi * np.outer(xs, k))  # (ncp, K)


def turbulence_store(levels: int = 4, coarsest: int = 2, micro: int = 65, degree: int = 3, K: int = 48,
                     seed: int = SEED, kmax: float = 12.0, ncp_range=(40, 65), progress=None, alloc=None):
    """(manifest, {addr: .mfa image}) of the config-3 synthetic turbulence model.

    alloc(total_bytes) -> uint8 array (e.g. a pinned host buffer); images are
    then zero-copy views into it, in sorted address order."""
    from .model import serialized_size

    man = skeleton(levels, coarsest, micro)
    man.degree = degree
    addrs = sorted(man.entries)
    sizes = [serialized_size(ncp_for(a, *ncp_range), degree) for a in addrs]
    total = int(sum(sizes))
    buf = alloc(total) if alloc is not None else np.empty(total, dtype=np.uint8)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    kvec, A = _modes(K, seed, kmax)
    # value range estimate for the [0.02, 0.98] normalization
    rng = np.random.default_rng(seed + 1)
    pts = rng.uniform(-1, 1, size=(1 << 15, 3))
    vals = np.real(np.exp(2j * np.pi * pts @ kvec.T) @ A)
    vmin, vmax = float(vals.min()), float(vals.max())
    scale = 0.96 / (vmax - vmin)
    offset = 0.02 - vmin * scale
    blobs = {}
    for n_done, addr in enumerate(addrs):
        ncp = ncp_for(addr, *ncp_range)
        P = fit_operator(micro, ncp, degree)
        ext = man.entries[addr].extent
        F = [_mode_factors(P, ext[a, 0], ext[a, 1], micro, kvec[:, a]) for a in range(3)]
        G = (F[1][:, None, :] * F[2][None, :, :]).reshape(ncp * ncp, K)
        ctrl = np.real((F[0] * A[None, :]) @ G.T).reshape(ncp, ncp, ncp)
        ctrl = ctrl * scale + offset  # the fit reproduces affine maps exactly
        view = buf[offs[n_done]:offs[n_done + 1]]
        view[:] = np.frombuffer(pack_mfa(degree, ctrl.astype(np.float32)), dtype=np.uint8)
        blobs[addr] = view
        ent = man.entries[addr]
        ent.ncp, ent.nbytes, ent.path, ent.is_complex = ncp, len(view), addr.file_name, True
        if progress and n_done % 500 == 0:
            progress(n_done, len(addrs))
    man.error_bound = None
    return man, blobs


def ml_value(x, y, z, f_m: float = 6.0, alpha: float = 0.05):
    """Marschner-Lobb field (Marschner & Lobb 1994), normalized to [0, 1]
    (the reference's volume.ml_value, float64, radius by np.hypot)."""
    x, y, z = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64), np.asarray(z, dtype=np.float64)
    r = np.hypot(x, y)
    rho = np.cos(2.0 * np.pi * f_m * np.cos(np.pi * r / 2.0))
    return (1.0 - np.sin(np.pi * z / 2.0) + alpha * (1.0 + rho)) / (2.0 * (1.0 + alpha))


def ml_volume(dims=(257, 257, 257), bounds=((0.0, 7.0),) * 3):
    """The reference's sample_grid(marschner_lobb(), dims) (volume.py:127-139):
    float32 samples [ix, iy, iz] over the inclusive bounds, with .bounds."""
    from types import SimpleNamespace

    b = np.asarray(bounds, dtype=np.float64)
    axes = [np.linspace(b[a, 0], b[a, 1], int(dims[a])) for a in range(3)]
    X, Y, Z = np.meshgrid(*axes, indexing="ij")
    return SimpleNamespace(samples=ml_value(X, Y, Z).astype(np.float32), bounds=b)


def field_store(levels: int, coarsest: int, micro: int, degree: int, ncp_of, fn=ml_value,
                bounds=((0.0, 7.0),) * 3):
    """Sample `fn` over physical `bounds` on every block's micro lattice and fit
    with ncp_of(addr) control points; returns (manifest, {addr: .mfa bytes})."""
    man = skeleton(levels, coarsest, micro, bounds)
    man.degree = degree
    b = np.asarray(bounds, dtype=np.float64)
    blobs = {}
    for addr in sorted(man.entries):
        ext = man.entries[addr].extent
        axes = [b[a, 0] + (ext[a] + 1.0) / 2.0 * (b[a, 1] - b[a, 0]) for a in range(3)]
        grids = [np.linspace(axes[a][0], axes[a][1], micro) for a in range(3)]
        X, Y, Z = np.meshgrid(*grids, indexing="ij")
        samples = fn(X, Y, Z).astype(np.float32).astype(np.float64)
        ncp = int(ncp_of(addr))
        P = fit_operator(micro, ncp, degree)
        c = np.einsum("ai,ijk->ajk", P, samples)
        c = np.einsum("bj,ajk->abk", P, c)
        c = np.einsum("ck,abk->abc", P, c)
        blob = pack_mfa(degree, c.astype(np.float32))
        blobs[addr] = blob
        ent = man.entries[addr]
        ent.ncp, ent.nbytes, ent.path = ncp, len(blob), addr.file_name
    return man, blobs


def turbulence_ds_blocks(addrs, levels: int = 4, coarsest: int = 2, micro: int = 65, ghost: int = 1, K: int = 48,
                         seed: int = SEED, kmax: float = 12.0):
    """{addr: DS block file image} of the same synthetic turbulence field as
    turbulence_store, sampled directly on each block's micro lattice plus the
    ghost layer (clamped at the volume faces, as downsample.build_ds_store),
    for the DS-vs-spline comparison (paper Fig. 15)."""
    import struct

    man = skeleton(levels, coarsest, micro)
    kvec, A = _modes(K, seed, kmax)
    rng = np.random.default_rng(seed + 1)
    pts = rng.uniform(-1, 1, size=(1 << 15, 3))
    vals = np.real(np.exp(2j * np.pi * pts @ kvec.T) @ A)
    vmin, vmax = float(vals.min()), float(vals.max())
    scale = 0.96 / (vmax - vmin)
    offset = 0.02 - vmin * scale
    out = {}
    for addr in addrs:
        ext = man.entries[addr].extent
        E = []
        for a in range(3):
            step = (ext[a, 1] - ext[a, 0]) / (micro - 1)
            xs = np.clip(ext[a, 0] + step * np.arange(-ghost, micro + ghost), -1.0, 1.0)
            E.append(np.exp(2j * np.pi * np.outer(xs, kvec[:, a])))  # (n, K)
        n = micro + 2 * ghost
        G = (E[1][:, None, :] * E[2][None, :, :]).reshape(n * n, -1)
        v = np.real((E[0] * A[None, :]) @ G.T).reshape(n, n, n) * scale + offset
        out[addr] = struct.pack("<4I", n, n, n, ghost) + v.astype("<f4").ravel(order="F").tobytes()
    return out
