"""Golden point queries of DS baseline blocks from the UNMODIFIED reference
(downsample.DsBlock.values_at / gradients_at, downsample.py:101-138).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_ds_points_golden.py

Output tests/golden/ds_points.npz: for ghost 0 and 1, three blocks of the
33^3 Marschner-Lobb DS store (2 levels, micro 9): samples, ghost, extent,
600 seeded world points around each block (some outside: clipped), values
and gradients."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import downsample  # noqa: E402
from splinecast.volume import marschner_lobb, sample_grid  # noqa: E402

OUT = Path(__file__).resolve().parent / "ds_points.npz"


def main():
    out = {}
    vol = sample_grid(marschner_lobb(), (33, 33, 33))
    rng = np.random.default_rng(7)
    k = 0
    for g in (0, 1):
        _, blocks = downsample.build_ds_store(vol, levels=2, micro_dims=9, coarsest=2, ghost=g)
        keys = sorted(blocks)
        for a in (keys[0], keys[len(keys) // 2], keys[-1]):
            b = blocks[a]
            lo, hi = b.extent[:, 0], b.extent[:, 1]
            span = hi - lo
            pts = lo + rng.uniform(-0.1, 1.1, size=(600, 3)) * span
            out[f"b{k}_samples"] = b.samples
            out[f"b{k}_ghost"] = np.array(b.ghost)
            out[f"b{k}_extent"] = b.extent
            out[f"b{k}_lod"] = np.array(a.lod)
            out[f"b{k}_points"] = pts
            out[f"b{k}_values"] = b.values_at(pts)
            out[f"b{k}_grads"] = b.gradients_at(pts)
            k += 1
    out["nblocks"] = np.array(k)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
