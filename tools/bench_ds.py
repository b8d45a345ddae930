"""DS baseline vs Adaptive-FAM on the config-3 geometry (paper Fig. 15):
1024^2 frames of the same synthetic turbulence field rendered from raw
ghosted DS blocks (trilinear) and from the spline store; device time per
frame (CUDA events), samples, and the bytes of the visible set."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, synth  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
frames = [3, 4, 5]
need = sorted({a for k in frames for a in render.select_visible(povs[k], man)})
ds_blobs = synth.turbulence_ds_blocks(need)
dsm = DeviceStore(len(need) + 1, 67)
ds_res = {a: dsm.load_ds(ds_blobs[a], man.entries[a].extent, a.lod) for a in need}
sps = DeviceStore(len(need) + 1, 65)
sp_res = {a: sps.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
torch.cuda.synchronize()
for kind, res, nbytes in (("ds", ds_res, {a: len(ds_blobs[a]) for a in need}),
                          ("spline", sp_res, {a: len(blobs[a]) for a in need})):
    ms, samples, vis_bytes = [], [], []
    for rep in range(2):
        for k in frames:
            vis = render.select_visible(povs[k], man)
            out, info, _ = render.render_part(povs[k], {a: res[a] for a in vis}, tf, params)
            if rep:
                ms.append(info["kernel_ms"])
                samples.append(info["samples"])
                vis_bytes.append(sum(nbytes[a] for a in vis))
    print(json.dumps({"blocks": kind, "frames": frames, "kernel_ms": float(np.mean(ms)),
                      "samples_per_frame": float(np.mean(samples)),
                      "samples_per_s": float(np.sum(samples) / (np.sum(ms) * 1e-3)),
                      "visible_bytes": float(np.mean(vis_bytes))}), flush=True)
