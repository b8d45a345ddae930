"""Diagnostic: K2 kernel time and sample-path counts on config-3 orbit frames."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2409_00184_b200 import render, runtime, synth
from paper_2409_00184_b200.device import DeviceStore

man, blobs = synth.turbulence_store()
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
ds = DeviceStore(len(blobs) + 1, 65)
res = {a: ds.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.environ.get("TAG", "")
for k in [0, 3, 3, 4, 5, 6]:
    vis = render.select_visible(povs[k], man)
    blocks = {a: res[a] for a in vis}
    flush.zero_()
    torch.cuda.synchronize()
    out, info, _ = render.render_part(povs[k], blocks, tf, params)
    print(tag, k, "kernel_ms %.3f" % info["kernel_ms"], "samples", info["samples"], "shaded", info["shaded_samples"],
          "exact", info.get("exact_samples"), "cells", info.get("exact_cells"), "fp64", info["fp64_samples"], flush=True)
