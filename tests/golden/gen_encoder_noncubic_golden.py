"""Golden vectors for the encoder on NON-CUBIC micro-blocks, from the
UNMODIFIED reference (bspline.fit_tensor_product fits any 3-D grid; the
search's NCP range runs up to samples.shape[0], encoder.py:104).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_encoder_noncubic_golden.py

Output tests/golden/encoder_noncubic.npz:
  fit_*        _fit_and_measure on a seeded (5, 9, 7) block, p = 2, every NCP
  search_*     in_level_search on it (full sweep and bisection)
  bad_msg      the ValueError of a (9, 9, 5) block's sweep (ncp 9 > 5 on axis 2)
  vol_*        encode_volume on a (9, 17, 17) volume, micro_dims (5, 9, 9),
               2 levels, coarsest 1, p = 2 adaptive
"""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import encoder  # noqa: E402
from splinecast.volume import ScalarVolume  # noqa: E402

OUT = Path(__file__).resolve().parent / "encoder_noncubic.npz"


def aniso_block(shape, seed):
    rng = np.random.default_rng(seed)
    axes = [np.linspace(0, 1, n) for n in shape]
    X, Y, Z = np.meshgrid(*axes, indexing="ij")
    v = np.zeros_like(X)
    for _ in range(4):
        k = rng.uniform(0.5, 3.0, 3)
        ph = rng.uniform(0, 2 * np.pi, 3)
        v += rng.uniform(0.1, 0.3) * np.sin(k[0] * np.pi * X + ph[0]) * np.cos(k[1] * np.pi * Y + ph[1]) * \
            np.sin(k[2] * np.pi * Z + ph[2])
    v += 0.02 * rng.standard_normal(v.shape)
    return (0.5 + v).astype(np.float32)


def main():
    out = {}
    s = aniso_block((5, 9, 7), 11)
    out["fit_samples"] = s
    rm = []
    for ncp in range(3, 6):
        mm, r = encoder._fit_and_measure(s, ncp, 2, ((-1, 1),) * 3, 1)
        out[f"fit_ctrl_{ncp}"] = mm.control
        rm.append(r)
    out["fit_rmse"] = np.array(rm)
    for k, (bound, mono) in enumerate([(3e-2, False), (3e-2, True)]):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = encoder.in_level_search(s, bound, 2, assume_monotone=mono)
        out[f"search_{k}_case"] = np.array([bound, float(mono)])
        out[f"search_{k}_star"] = np.array([r.ncp_star, int(r.met_bound), int(r.is_complex)])
        out[f"search_{k}_profile"] = np.array(sorted(r.profile.rmse_by_ncp.items()), dtype=np.float64)
        out[f"search_{k}_ctrl"] = r.model.control
    try:
        encoder.in_level_search(aniso_block((9, 9, 5), 12), 1e-2, 2)
        out["bad_msg"] = np.array("")
    except ValueError as exc:
        out["bad_msg"] = np.array(str(exc))
    vol = ScalarVolume(samples=aniso_block((9, 17, 17), 13), bounds=np.array([[-1.0, 1.0]] * 3))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        man, models, stats = encoder.encode_volume(vol, levels=2, micro_dims=(5, 9, 9), degree=2, error_bound=3e-2,
                                                   coarsest=1, mode="adaptive")
    addrs = sorted(man.entries)
    out["vol_samples"] = vol.samples
    out["vol_addr"] = np.array([(a.lod, *a.ijk) for a in addrs], dtype=np.int64)
    out["vol_ncp"] = np.array([man.entries[a].ncp for a in addrs], dtype=np.int64)
    out["vol_complex"] = np.array([int(man.entries[a].is_complex) for a in addrs], dtype=np.int64)
    out["vol_stats"] = np.array([stats.total_blocks, stats.searched_blocks, len(stats.unmet_blocks)])
    for i, a in enumerate(addrs):
        out[f"vol_ctrl_{i}"] = models[a].control
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes", "bad_msg:", out["bad_msg"])


if __name__ == "__main__":
    main()
