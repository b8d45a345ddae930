"""Golden vectors for the down-sampled (DS) baseline, from the UNMODIFIED
reference (downsample.py + render.py).

Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_ds_golden.py

Output tests/golden/ds.npz:
  store_g<g>_*   DS stores (ghost g = 0, 1) of a 33^3 Marschner-Lobb volume,
                 2 levels of 9^3 blocks: manifest JSON, block keys, the .dsb
                 bytes (serialize_ds) concatenated with offsets
  <frame>_*      render() frames of those stores (rgba, sample count, pov,
                 params, tf, visible list)
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from splinecast import downsample, render  # noqa: E402
from splinecast.volume import marschner_lobb, sample_grid  # noqa: E402

OUT = Path(__file__).resolve().parent / "ds.npz"


class Counting:
    def __init__(self, block, counter):
        self.b, self.c = block, counter
        self.extent, self.lod = block.extent, block.lod

    def values_at(self, pts):
        self.c[0] += len(pts)
        return self.b.values_at(pts)

    def gradients_at(self, pts):
        return self.b.gradients_at(pts)


def main():
    out = {}
    vol = sample_grid(marschner_lobb(), (33, 33, 33))
    stores = {}
    for g in (0, 1):
        man, blocks = downsample.build_ds_store(vol, levels=2, micro_dims=9, coarsest=2, ghost=g)
        keys = sorted(blocks)
        blobs = [downsample.serialize_ds(blocks[a]) for a in keys]
        for a, b in zip(keys, blobs):
            man.entries[a].path = a.file_name.replace(".mfa", ".dsb")
            man.entries[a].nbytes = len(b)
        out[f"store_g{g}_manifest"] = np.frombuffer(json.dumps(man.to_json()).encode(), dtype=np.uint8)
        out[f"store_g{g}_keys"] = np.array([a.key for a in keys])
        out[f"store_g{g}_offsets"] = np.concatenate([[0], np.cumsum([len(b) for b in blobs])]).astype(np.int64)
        out[f"store_g{g}_blob"] = np.frombuffer(b"".join(blobs), dtype=np.uint8)
        stores[g] = (man, blocks)
    tf = render.TransferFunction.ml_preset()
    P = render.PointOfView
    jobs = [
        ("ds1_a", 1, P([0.4, 0.3, 2.0], [-0.1, -0.1, -1.0], [0, 1, 0]), render.RenderParams(32, 32, 0.01)),
        ("ds1_b", 1, P([2.0, 1.6, 2.6], [-0.55, -0.44, -0.71], [0, 1, 0], 50.0),
         render.RenderParams(width=40, height=24, sample_distance=0.008, o_max=1.0)),
        ("ds0_a", 0, P([0.4, 0.3, 2.0], [-0.1, -0.1, -1.0], [0, 1, 0]), render.RenderParams(32, 32, 0.01)),
        ("ds0_c", 0, P([0.5, 0.5, 1.1], [0, 0, -1], [0, 1, 0], 60.0),
         render.RenderParams(width=24, height=24, sample_distance=0.005, reference_step=0.01)),
    ]
    names = []
    for name, g, pov, params in jobs:
        man, blocks = stores[g]
        vis = render.select_visible(pov, man, params.aspect)
        counter = [0]
        resident = {a: Counting(blocks[a], counter) for a in vis}
        t = time.time()
        fr = render.render(pov, resident, tf, params)
        print(f"frame {name}: {counter[0]} samples {time.time() - t:.1f}s", flush=True)
        out[f"{name}_rgba"] = fr.rgba
        out[f"{name}_samples"] = np.array(counter[0])
        out[f"{name}_ghost"] = np.array(g)
        out[f"{name}_pov"] = np.array([*pov.position, *pov.direction, *pov.up, pov.fov_y])
        out[f"{name}_params"] = np.array([params.width, params.height, params.sample_distance, params.o_max,
                                          params.reference_step if params.reference_step is not None else np.nan,
                                          params.near, params.ambient, params.diffuse, params.specular,
                                          params.shininess])
        out[f"{name}_vis"] = np.array([(a.lod, *a.ijk) for a in vis], dtype=np.int32)
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
