"""Where does caching_ms go in the e2e replay (visibility, cache fetches incl.
uploads, loader sync)?"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, tiles  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
ds = DeviceStore(201, 65)
loader = runtime.make_loader(None, man, ds, source=lambda a: blobs[a])
cache = runtime.ModelCache(200, loader)
T = {"vis": [], "fetch": [], "sync": [], "loads": []}
orig_cf = runtime.cache_frame


def cache_frame(pov, manifest, cache_, aspect=1.0):
    t0 = time.perf_counter()
    visible = render.select_visible(pov, manifest, aspect)
    t1 = time.perf_counter()
    cache_.begin_frame(visible)
    m0 = cache_.misses
    resident = cache_.fetch_many(visible)
    t2 = time.perf_counter()
    cache_._loader.sync()
    t3 = time.perf_counter()
    T["vis"].append((t1 - t0) * 1e3)
    T["fetch"].append((t2 - t1) * 1e3)
    T["sync"].append((t3 - t2) * 1e3)
    T["loads"].append(cache_.misses - m0)
    return resident


runtime.cache_frame = cache_frame


def draw(pov, resident, tf_, params_):
    return tiles.render_tiles(pov, resident, tf_, params_, band_rows=8)


runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
for k in T:
    T[k].clear()
_, _, agg = runtime.replay(povs[3:43], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
print({k: round(v, 3) if isinstance(v, float) else v for k, v in agg.items()})
print({k: round(float(np.mean(v)), 4) for k, v in T.items()})
