"""Golden vectors for the encoder inner loop, from the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_encoder_golden.py

Output tests/golden/encoder.npz:
  fit_<c>_*        model.fit + encoder.error_rmse (encoder._fit_and_measure)
                   on seeded blocks: control points (float32) and RMSE per NCP
  search_<c>_*     encoder.in_level_search (full sweep and bisection):
                   ncp_star, met_bound, is_complex, the RMSE profile
  vol_<d>_*        encoder.encode_volume on a 33^3 Marschner-Lobb volume
                   (2 levels of 9^3 micro-blocks, adaptive; p=2 full sweep,
                   p=3 bisection): per-block NCP,
                   complexity, stats, and the control points of every block
"""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import encoder, model  # noqa: E402
from splinecast.volume import marschner_lobb, sample_grid  # noqa: E402

OUT = Path(__file__).resolve().parent / "encoder.npz"


def smooth_block(m, seed):
    rng = np.random.default_rng(seed)
    x = np.linspace(0, 1, m)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    v = np.zeros_like(X)
    for _ in range(4):
        k = rng.uniform(0.5, 3.0, 3)
        ph = rng.uniform(0, 2 * np.pi, 3)
        v += rng.uniform(0.1, 0.3) * np.sin(k[0] * np.pi * X + ph[0]) * np.cos(k[1] * np.pi * Y + ph[1]) * \
            np.sin(k[2] * np.pi * Z + ph[2])
    v += 0.02 * rng.standard_normal(v.shape)  # texture so small NCPs miss the bound
    return (0.5 + v).astype(np.float32)


def main():
    out = {}
    # --- _fit_and_measure on seeded blocks (every NCP)
    fit_cases = [(9, 2, 1), (9, 3, 2), (17, 2, 3), (17, 3, 4), (13, 1, 5)]
    out["fit_cases"] = np.array(fit_cases, dtype=np.int64)
    for c, (m, deg, seed) in enumerate(fit_cases):
        s = smooth_block(m, seed)
        out[f"fit_{c}_samples"] = s
        rm = []
        for ncp in range(deg + 1, m + 1):
            mm, r = encoder._fit_and_measure(s, ncp, deg, ((-1, 1),) * 3, 1)
            out[f"fit_{c}_ctrl_{ncp}"] = mm.control
            rm.append(r)
        out[f"fit_{c}_rmse"] = np.array(rm)
    # --- in_level_search
    search_cases = [(0, 2e-2, False), (0, 2e-2, True), (2, 1.5e-2, False), (3, 1.5e-2, True), (3, 1e-9, False),
                    (4, 3e-2, False)]
    out["search_cases"] = np.array([(c, b, mono) for c, b, mono in search_cases], dtype=np.float64)
    for k, (c, bound, mono) in enumerate(search_cases):
        m, deg, seed = fit_cases[c]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = encoder.in_level_search(out[f"fit_{c}_samples"], bound, deg, assume_monotone=mono)
        out[f"search_{k}_star"] = np.array([r.ncp_star, int(r.met_bound), int(r.is_complex)])
        prof = sorted(r.profile.rmse_by_ncp.items())
        out[f"search_{k}_profile"] = np.array(prof, dtype=np.float64)
        out[f"search_{k}_ctrl"] = r.model.control
    # --- encode_volume (adaptive, 2 levels, micro 9, 33^3 Marschner-Lobb)
    vol = sample_grid(marschner_lobb(), (33, 33, 33))
    vol_cases = {2: (5e-2, False), 3: (2e-2, True)}  # degree: (error bound, assume_monotone)
    for deg, (bound, mono) in vol_cases.items():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            man, models, stats = encoder.encode_volume(vol, levels=2, micro_dims=9, degree=deg, error_bound=bound,
                                                       coarsest=2, mode="adaptive", assume_monotone=mono)
        out[f"vol_{deg}_case"] = np.array([bound, float(mono)])
        addrs = sorted(man.entries)
        out[f"vol_{deg}_addr"] = np.array([(a.lod, *a.ijk) for a in addrs], dtype=np.int64)
        out[f"vol_{deg}_ncp"] = np.array([man.entries[a].ncp for a in addrs], dtype=np.int64)
        out[f"vol_{deg}_complex"] = np.array([int(man.entries[a].is_complex) for a in addrs], dtype=np.int64)
        out[f"vol_{deg}_stats"] = np.array([stats.total_blocks, stats.searched_blocks, len(stats.unmet_blocks)])
        for i, a in enumerate(addrs):
            out[f"vol_{deg}_ctrl_{i}"] = models[a].control
    out["vol_samples"] = vol.samples
    out["vol_bounds"] = vol.bounds
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
