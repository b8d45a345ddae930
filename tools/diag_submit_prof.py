"""Host time of render.submit on resident config-3 blocks, by function."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
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
for k in range(3):
    render.render(povs[3 + k], frames[k], tf, params)
torch.cuda.synchronize()
ts = []
pr = cProfile.Profile()
for k in range(20):
    pr.enable()
    t0 = time.perf_counter()
    p = render.submit(povs[3 + k], frames[k], tf, params)
    ts.append((time.perf_counter() - t0) * 1e3)
    pr.disable()
    p.result()
ts.sort()
print("submit host ms: median %.3f min %.3f" % (ts[10], ts[0]))
pstats.Stats(pr).sort_stats("cumtime").print_stats(22)
