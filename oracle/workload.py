"""Product-free inputs of the CPU reference arm (bench.py --impl reference).

TEST INFRASTRUCTURE ONLY, like the rest of oracle/: numpy and the oracle
library, never the product package, so the reference arm maps no libafam
code.  It restates, independently of paper_2409_00184_b200.synth:

* the config-3 model (1024^3-equivalent synthetic turbulence, 4 LODs,
  coarsest 2, micro 65 -> 4,680 blocks, degree 3): per-block NCP from the
  blake2b hash of the block key in [40, 65], the endpoint-pinned
  least-squares fit operator of the reference encoder (bspline.py:109-159)
  applied mode by mode, FORMAT.md .mfa images -- byte-identical to the
  product's synthesis (tests/test_bench_contract.py checks it);
* the LOD skeleton's dyadic block extents (reference partition.py:229-233);
* the .mfa reader (reference model.py:121-148, FORMAT.md:16-70);
* orbit_trajectory (reference runtime.py:350-361), PointOfView's
  normalisation (render.py:52-66), RenderParams' defaults (render.py:168-192)
  and TransferFunction.ml_preset (render.py:148-165) as plain namespaces.
"""

from __future__ import annotations

import hashlib
from functools import lru_cache
from types import SimpleNamespace
from typing import NamedTuple

import numpy as np

SEED = 20261017


class Addr(NamedTuple):
    lod: int
    ijk: tuple

    @property
    def key(self) -> str:
        return "%d/%d_%d_%d" % (self.lod, *self.ijk)


def clamped_knots(ncp: int, degree: int) -> np.ndarray:
    """Clamped uniform knot vector (reference bspline.py:29-38): interior k/nspan."""
    interior = np.arange(1, ncp - degree, dtype=np.float64) / (ncp - degree)
    return np.concatenate([np.zeros(degree + 1), interior, np.ones(degree + 1)])


def _basis_rows(params, knots, ncp, degree):
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
    B[np.arange(n)[:, None], span[:, None] - degree + np.arange(degree + 1)[None, :]] = vals
    return B


@lru_cache(maxsize=256)
def fit_operator(m: int, ncp: int, degree: int) -> np.ndarray:
    """(ncp, m): uniform samples -> endpoint-pinned least-squares coefficients."""
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


def ncp_for(addr: Addr, lo: int = 40, hi: int = 65) -> int:
    h = int.from_bytes(hashlib.blake2b(addr.key.encode(), digest_size=4).digest(), "little")
    return hi - h % (hi - lo + 1)


def pack_mfa(degree: int, control: np.ndarray) -> bytes:
    ncp = control.shape[0]
    kv = clamped_knots(ncp, degree).astype("<f4")
    return bytes([degree]) + kv[1:].tobytes() * 3 + np.asarray(control, dtype="<f4").ravel(order="F").tobytes()


def serialized_size(ncp: int, degree: int) -> int:
    return 1 + ((ncp + degree) * 3 + ncp ** 3) * 4


def block_extent(ijk, bpa: int) -> np.ndarray:
    idx = np.asarray(ijk, dtype=np.float64)
    return np.stack([2.0 * (idx / bpa) - 1.0, 2.0 * ((idx + 1.0) / bpa) - 1.0], axis=1)


def skeleton(levels: int, coarsest: int, micro: int):
    """Manifest namespace (levels, finest_blocks_per_axis, micro_dims,
    entries[Addr] -> .extent/.ncp) of a (levels, coarsest, micro) hierarchy."""
    finest = coarsest << (levels - 1)
    entries = {}
    for lod in range(1, levels + 1):
        b = coarsest << (levels - lod)
        for i in range(b):
            for j in range(b):
                for k in range(b):
                    entries[Addr(lod, (i, j, k))] = SimpleNamespace(extent=block_extent((i, j, k), b), ncp=None)
    return SimpleNamespace(levels=levels, finest_blocks_per_axis=finest, micro_dims=(micro,) * 3, entries=entries)


def _modes(K: int, seed: int, kmax: float):
    rng = np.random.default_rng(seed)
    dirs = rng.normal(size=(K, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    kmag = np.exp(rng.uniform(np.log(1.0), np.log(kmax), size=K))
    kvec = dirs * kmag[:, None]
    amp = kmag ** (-5.0 / 3.0)
    phase = rng.uniform(0, 2 * np.pi, size=K)
    return kvec, amp * np.exp(1j * phase)


def turbulence_store(levels: int = 4, coarsest: int = 2, micro: int = 65, degree: int = 3, K: int = 48,
                     seed: int = SEED, kmax: float = 12.0, ncp_range=(40, 65), addrs=None):
    """(manifest namespace, {Addr: .mfa bytes}) of the config-3 model; with
    `addrs`, only those blocks' images are synthesised."""
    man = skeleton(levels, coarsest, micro)
    kvec, A = _modes(K, seed, kmax)
    rng = np.random.default_rng(seed + 1)
    pts = rng.uniform(-1, 1, size=(1 << 15, 3))
    vals = np.real(np.exp(2j * np.pi * pts @ kvec.T) @ A)
    vmin, vmax = float(vals.min()), float(vals.max())
    scale = 0.96 / (vmax - vmin)
    offset = 0.02 - vmin * scale
    for a, e in man.entries.items():
        e.ncp = ncp_for(a, *ncp_range)
    want = sorted(man.entries) if addrs is None else sorted(addrs)
    blobs = {}
    for a in want:
        ncp = man.entries[a].ncp
        P = fit_operator(micro, ncp, degree)
        ext = man.entries[a].extent
        F = []
        for ax in range(3):
            xs = ext[ax, 0] + (ext[ax, 1] - ext[ax, 0]) * (np.arange(micro) / (micro - 1))
            F.append(P @ np.exp(2j * np.pi * np.outer(xs, kvec[:, ax])))
        G = (F[1][:, None, :] * F[2][None, :, :]).reshape(ncp * ncp, K)
        ctrl = np.real((F[0] * A[None, :]) @ G.T).reshape(ncp, ncp, ncp) * scale + offset
        blobs[a] = pack_mfa(degree, ctrl.astype(np.float32))
    return man, blobs


def parse_mfa(data: bytes, ncp: int, extent, lod: int = 1):
    """model.deserialize (model.py:121-148): [u8 d][3*(ncp+d) f32 knots t1..][ncp^3 f32, x fastest]."""
    d = data[0]
    stored = ncp + d
    if len(data) != 1 + (stored * 3 + ncp ** 3) * 4:
        raise ValueError("model length mismatch")
    knots = np.zeros((3, stored + 1), dtype=np.float32)
    off = 1
    for a in range(3):
        knots[a, 1:] = np.frombuffer(data, dtype="<f4", count=stored, offset=off)
        off += stored * 4
    ctrl = np.frombuffer(data, dtype="<f4", count=ncp ** 3, offset=off).reshape((ncp,) * 3, order="F")
    return SimpleNamespace(degree=int(d), knots=knots, control=ctrl,
                           extent=np.asarray(extent, dtype=np.float64).reshape(3, 2), lod=lod)


def point_of_view(position, direction, up, fov_y: float = 45.0):
    """PointOfView (render.py:52-66): the direction stored normalised."""
    d = np.asarray(direction, dtype=np.float64).reshape(3)
    return SimpleNamespace(position=np.asarray(position, dtype=np.float64).reshape(3), direction=d / np.linalg.norm(d),
                           up=np.asarray(up, dtype=np.float64).reshape(3), fov_y=float(fov_y))


def orbit_trajectory(count: int, radius: float = 3.0, center=(0.0, 0.0, 0.0), fov_y: float = 45.0) -> list:
    c = np.asarray(center, dtype=np.float64)
    povs = []
    for k in range(count):
        ang = 2.0 * np.pi * k / count
        pos = c + np.array([np.sin(ang), 0.0, np.cos(ang)]) * radius
        d = c - pos
        d /= np.linalg.norm(d)
        povs.append(point_of_view(pos, d, [0.0, 1.0, 0.0], fov_y))
    return povs


def render_params(width: int = 512, height: int = 512, sample_distance: float = 1e-3, o_max: float = 0.99):
    return SimpleNamespace(width=width, height=height, sample_distance=sample_distance, o_max=o_max,
                           reference_step=None, near=1e-3, ambient=0.1, diffuse=0.7, specular=0.2, shininess=32.0,
                           aspect=width / height)


def ml_preset():
    color = [[0.00, 0.10, 0.15, 0.60], [0.35, 0.20, 0.55, 0.85], [0.50, 0.95, 0.95, 0.90],
             [0.65, 0.95, 0.55, 0.15], [1.00, 0.80, 0.20, 0.10]]
    alpha = [[0.00, 0.0], [0.38, 0.0], [0.50, 0.35], [0.62, 0.0], [1.00, 0.0]]
    return SimpleNamespace(color_points=np.array(color), opacity_points=np.array(alpha), domain=(0.0, 1.0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or platform.machine()
