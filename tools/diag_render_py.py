"""cProfile of the host side of tiles.render_tiles (blocks resident)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, tiles  # noqa: E402
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
    tiles.render_tiles(povs[3 + k], frames[k], tf, params)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for k in range(20):
    tiles.render_tiles(povs[3 + k], frames[k], tf, params)
pr.disable()
print("per frame %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
