"""Diagnostic: golden frames through render() — PSNR, sample/shade/exact counts."""
import os, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from helpers import npz, golden_store, params_ns, tf_ns, pov_ns
from oracle import oracle
from paper_2409_00184_b200 import render
from paper_2409_00184_b200.partition import BlockAddress
from test_gpu_parity import _to_product

z = npz("frames.npz")
for name in list(z["names"]):
    man, models, _ = golden_store(str(z[f"{name}_store"]))
    pm = _to_product(models)
    vis = [tuple(int(v) for v in r) for r in z[f"{name}_vis"]]
    resident = {BlockAddress(v[0], v[1:]): pm[BlockAddress(v[0], v[1:])] for v in vis}
    p = params_ns(z[f"{name}_params"])
    params = render.RenderParams(width=p.width, height=p.height, sample_distance=p.sample_distance, o_max=p.o_max,
                                 reference_step=p.reference_step, near=p.near, ambient=p.ambient,
                                 diffuse=p.diffuse, specular=p.specular, shininess=p.shininess)
    t = tf_ns(z[f"{name}_tf"])
    tf = render.TransferFunction(t.color_points, t.opacity_points, t.domain)
    frame = render.render(pov_ns(z[f"{name}_pov"]), resident, tf, params)
    want = z[f"{name}_rgba"]
    st = render.render.last_stats
    d = np.abs(frame.rgba.astype(int) - want.astype(int))
    print(name, "psnr %.2f" % oracle.psnr(frame.rgba, want), "maxdiff", d.max(axis=(0, 1)).tolist(),
          "samples", st["samples"], int(z[f"{name}_samples"]), "shaded", st["shaded_samples"],
          "exact", st["exact_samples"], "fp64", st["fp64_samples"], flush=True)
