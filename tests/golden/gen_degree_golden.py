"""Golden vectors for degrees above 3 from the UNMODIFIED reference (splinecast).

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/gen_degree_golden.py

The reference takes any degree (bspline.py:29-38, FORMAT.md "1 <= d < ncp");
the device path evaluates degrees 1..AFAM_MAX_DEGREE (15), degrees above 3
through a float64 Cox-de Boor path.  These fixtures pin the oracle and that
path: evaluate_points[_with_gradient] (degrees 4, 5, 7; clamped-uniform and
non-uniform knots), decode_tensor_product (degrees 4, 6), a store encoded by
the reference's adaptive encoder at degree 5, and frames rendered from it.

Output: tests/golden/degree.npz, tests/golden/store_ml33_p5.npz
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

from splinecast import bspline, render  # noqa: E402
from splinecast.encoder import encode_volume  # noqa: E402
from splinecast.volume import marschner_lobb, sample_grid  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent))
from gen_golden import Counting, pack_store  # noqa: E402

OUT = Path(__file__).resolve().parent


def gen_points(out):
    rng = np.random.default_rng(20261018)
    cases = [(4, 9, False), (5, 10, False), (7, 12, False), (4, 11, True), (6, 8, True)]
    for ci, (degree, ncp, nonuniform) in enumerate(cases):
        coeff = rng.normal(size=(ncp, ncp, ncp)).astype(np.float32)
        kv = bspline.clamped_knots(ncp, degree)
        if nonuniform:  # strictly increasing interior knots, clamped ends
            inner = np.sort(rng.uniform(0.05, 0.95, ncp - degree - 1))
            kv = np.r_[np.zeros(degree + 1), inner, np.ones(degree + 1)]
        k32 = np.repeat(kv.astype(np.float32)[None, :], 3, axis=0)
        u = rng.uniform(0, 1, size=(400, 3))
        edge = [0.0, 1.0, -0.2, 1.3] + [float(x) for x in k32[0, degree:ncp + 1]]
        e = np.array([[a, edge[(i + 1) % len(edge)], edge[(i + 2) % len(edge)]] for i, a in enumerate(edge)])
        u = np.vstack([u, e])
        v, g = bspline.evaluate_points_with_gradient(coeff, degree, u, knots=tuple(k32.astype(np.float64)))
        out[f"p{ci}_degree"] = np.array(degree)
        out[f"p{ci}_coeff"] = coeff
        out[f"p{ci}_knots32"] = k32
        out[f"p{ci}_u"] = u
        out[f"p{ci}_v"] = v
        out[f"p{ci}_g"] = g
    out["npoints"] = np.array(len(cases))
    dcases = [(4, 9, 13), (6, 11, 9), (5, 7, 17)]
    for ci, (degree, ncp, m) in enumerate(dcases):
        coeff = rng.normal(size=(ncp, ncp, ncp)).astype(np.float32)
        out[f"d{ci}_degree"] = np.array(degree)
        out[f"d{ci}_coeff"] = coeff
        out[f"d{ci}_m"] = np.array(m)
        out[f"d{ci}_grid"] = bspline.decode_tensor_product(coeff.astype(np.float64), degree, (m, m, m))
    out["ndecode"] = np.array(len(dcases))


def gen_store_and_frames(out):
    t = time.time()
    vol = sample_grid(marschner_lobb(), (33, 33, 33))
    man, models, _ = encode_volume(vol, levels=2, micro_dims=17, degree=5, error_bound=2e-2, coarsest=1)
    print(f"ml33_p5: {len(models)} blocks, ncp {sorted({m.control.shape[0] for m in models.values()})} "
          f"{time.time() - t:.1f}s", flush=True)
    np.savez_compressed(OUT / "store_ml33_p5.npz", **pack_store(man, models))
    P = render.PointOfView
    tf = render.TransferFunction.ml_preset()
    jobs = [("a", P([0.6, 0.5, 1.2], [-0.6, -0.5, -1.2], [0, 1, 0]),
             render.RenderParams(width=32, height=32, sample_distance=0.01, o_max=1.0)),
            ("b", P([0.1, -0.2, 1.6], [0.05, 0.1, -1.0], [0, 1, 0], 70.0),
             render.RenderParams(width=28, height=24, sample_distance=0.008))]
    for name, pov, params in jobs:
        vis = render.select_visible(pov, man, params.aspect)
        counter = [0]
        resident = {a: Counting(models[a], counter) for a in vis}
        t = time.time()
        fr = render.render(pov, resident, tf, params)
        print(f"frame {name}: {counter[0]} samples {time.time() - t:.1f}s", flush=True)
        out[f"f{name}_rgba"] = fr.rgba
        out[f"f{name}_samples"] = np.array(counter[0])
        out[f"f{name}_pov"] = np.array([*pov.position, *pov.direction, *pov.up, pov.fov_y])
        out[f"f{name}_params"] = np.array([params.width, params.height, params.sample_distance, params.o_max,
                                           params.reference_step if params.reference_step is not None else np.nan,
                                           params.near, params.ambient, params.diffuse, params.specular,
                                           params.shininess])
        out[f"f{name}_tf"] = np.frombuffer(json.dumps(tf.to_json()).encode(), dtype=np.uint8)
        out[f"f{name}_vis"] = np.array([(a.lod, *a.ijk) for a in vis], dtype=np.int32)
    out["frames"] = np.array([j[0] for j in jobs])


def main():
    out = {}
    gen_points(out)
    gen_store_and_frames(out)
    np.savez_compressed(OUT / "degree.npz", **out)
    print("wrote", OUT / "degree.npz")


if __name__ == "__main__":
    main()
