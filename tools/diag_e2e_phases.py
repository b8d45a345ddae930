"""Per-phase host time of the e2e replay loop (cache_frame, submit, prefetch,
result) on the bench's config-4 setup, replicating runtime.replay's
submit path with timers."""
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
cache = runtime.ModelCache(200, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
ph = {k: [] for k in ("cache", "submit", "prefetch", "result", "kernel", "frame")}
for i, pov in enumerate(povs[:43]):
    t0 = time.perf_counter()
    resident = runtime.cache_frame(pov, man, cache, params.aspect)
    t1 = time.perf_counter()
    pend = tiles.submit_tiles(pov, resident, tf, params, band_rows=8)
    t2 = time.perf_counter()
    hist = list(povs[max(0, i - 7): i + 1])
    if "nopf" not in sys.argv:
        runtime.prefetch_loop(hist, man, cache, runtime._Done(pend), runtime.predict_next_linear, params.aspect)
    t3 = time.perf_counter()
    pend.result()
    t4 = time.perf_counter()
    if i >= 3:
        for k, v in zip(("cache", "submit", "prefetch", "result", "frame"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            ph[k].append(v * 1e3)
        ph["kernel"].append(tiles.render_tiles.last_stats["kernel_ms"])
print(" ".join("%s %.3f" % (k, np.median(v)) for k, v in ph.items()))
