"""Golden decisions of BASELINE config 2, from the UNMODIFIED reference encoder.

Run in the build container only (the reference is not on the GPU box; the
encode takes ~7 min on the CPU):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_config2_golden.py

Config 2: the Marschner-Lobb field sampled on 257^3
(volume.sample_grid), encoder.encode_volume(levels=2, micro_dims=65,
coarsest=2, degree=3, error_bound=1e-3, mode="adaptive").  The 29 MB store
is too large to commit; the GPU test re-encodes the same volume with the
B200 encoder and is pinned here to the reference's per-block NCP and
complexity decisions and to a strided subset of every block's float32
control points (within 1 ulp).

Output tests/golden/config2.npz:
  addr (72, 4)      (lod, i, j, k) in sorted order
  ncp, complex      per block
  ctrl_sub_<i>      models[addr].control[::8, ::8, ::8] (float32)
  maxabs            max |control| per block (the ill-conditioned ncp 64/65 blocks)
"""

from __future__ import annotations

import sys
import time
import warnings
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import encoder  # noqa: E402
from splinecast.volume import marschner_lobb, sample_grid  # noqa: E402

OUT = Path(__file__).resolve().parent / "config2.npz"


def main():
    vol = sample_grid(marschner_lobb(), (257, 257, 257))
    t0 = time.time()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        man, models, stats = encoder.encode_volume(vol, levels=2, micro_dims=65, degree=3, error_bound=1e-3,
                                                   coarsest=2, mode="adaptive")
    el = time.time() - t0
    addrs = sorted(man.entries)
    out = {
        "addr": np.array([(a.lod, *a.ijk) for a in addrs], dtype=np.int64),
        "ncp": np.array([man.entries[a].ncp for a in addrs], dtype=np.int64),
        "complex": np.array([int(man.entries[a].is_complex) for a in addrs], dtype=np.int64),
        "maxabs": np.array([float(np.abs(models[a].control).max()) for a in addrs]),
        "stats": np.array([stats.total_blocks, stats.searched_blocks, len(stats.unmet_blocks)]),
        "encode_s": np.array(el),
    }
    for i, a in enumerate(addrs):
        out[f"ctrl_sub_{i}"] = models[a].control[::8, ::8, ::8].copy()
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes; encode", round(el, 1), "s; ncp", out["ncp"].tolist())


if __name__ == "__main__":
    main()
