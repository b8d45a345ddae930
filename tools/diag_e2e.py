"""cProfile of the e2e replay loop (host overhead per frame)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
ds = DeviceStore(201, 65)
cache = runtime.ModelCache(200, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
kms = []


def draw(pov, resident, tf_, params_):
    out, info, _ = render.render_part(pov, resident, tf_, params_, band_rows=8)
    kms.append(info["kernel_ms"])
    return out.cpu().numpy()


runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
for mode in ("off", "linear"):
    kms.clear()
    pr = cProfile.Profile()
    pr.enable()
    t, _, agg = runtime.replay(povs[3:23], man, cache, tf, params, prefetch=mode, keep_frames=False, render_fn=draw)
    pr.disable()
    print(mode, agg, "kernel_ms mean", sum(kms) / len(kms))
    pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
