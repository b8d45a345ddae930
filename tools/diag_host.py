"""Where does a bench step's time go?  host prep vs kernel vs sync."""
import sys
import time

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
ds = DeviceStore(len(blobs) + 1, 65)
res = {a: ds.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty((1024, 1024, 4), dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
for mode in ("noflush", "flush", "flush+sleep"):
    rows = []
    for k in range(3, 13):
        pov = povs[k]
        t0 = time.perf_counter()
        vis = render.select_visible(pov, man)
        blocks = {a: res[a] for a in vis}
        t1 = time.perf_counter()
        if mode != "noflush":
            flush.zero_()
        if mode == "flush+sleep":
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t2 = time.perf_counter()
        _, info, _ = render.render_part(pov, blocks, tf, params, band_rows=8, out=out)
        t3 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        rows.append(((t1 - t0) * 1e3, (t3 - t2) * 1e3, e0.elapsed_time(e1)))
    r = np.array(rows)
    print(mode, "select %.2f ms | render_part wall %.2f ms | event %.2f ms" % tuple(r.mean(axis=0)), flush=True)
