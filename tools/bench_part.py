"""K2 time of one part of a frame split into `nparts` interleaved 8-row
bands (what each rank renders at N = nparts), blocks resident."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

plist = [int(v) for v in sys.argv[1:]] or [8]
man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
need = sorted({a for k in range(3, 23) for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
frames = [{a: res[a] for a in render.select_visible(povs[k], man)} for k in range(3, 23)]
for nparts in plist:
    for part in sorted({0, nparts - 1}):
        ks = []
        for rep in range(2):
            for k in range(20):
                _, info, _ = render.render_part(povs[3 + k], frames[k], tf, params, band_rows=8, nparts=nparts,
                                                part=part)
                if rep:
                    ks.append(info["kernel_ms"])
        print(f"  part {part}/{nparts}: kernel ms {np.mean(ks):.4f}", flush=True)
