"""K2 kernel time writing the frame to pinned host memory (zero-copy,
host_out) vs to device memory, same frames, blocks resident."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
need = sorted({a for k in range(3, 23) for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
frames = [{a: res[a] for a in render.select_visible(povs[k], man)} for k in range(3, 23)]
for rep in range(2):
    for mode in ("device", "host_out"):
        ks = []
        for k in range(20):
            _, info, _ = render.render_part(povs[3 + k], frames[k], tf, params, host_out=(mode == "host_out"))
            ks.append(info["kernel_ms"])
        print(mode, "kernel ms median %.3f mean %.3f" % (np.median(ks), np.mean(ks)))
