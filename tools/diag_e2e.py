"""Host overhead of the e2e replay loop: per-frame caching/rendering wall
time vs the render kernel's device time, prefetch off vs linear, plus a
cProfile of the rendering call."""
import cProfile
import pstats
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
rec = []
import threading  # noqa: E402
from paper_2409_00184_b200 import _lib  # noqa: E402

main = threading.main_thread()
lib = _lib.lib()
orig = lib.afam_render
T = {"c_call": [], "sync": [], "sync_other": []}


class Wrap:
    def __call__(self, *a):
        t0 = time.perf_counter()
        r = orig(*a)
        T["c_call"].append((time.perf_counter() - t0) * 1e3)
        return r


lib.afam_render = Wrap()
orig_sync = torch.cuda.Stream.synchronize


def sync(self):
    t0 = time.perf_counter()
    orig_sync(self)
    T["sync" if threading.current_thread() is main else "sync_other"].append((time.perf_counter() - t0) * 1e3)


torch.cuda.Stream.synchronize = sync


def draw(pov, resident, tf_, params_):
    t0 = time.perf_counter()
    fr = tiles.render_tiles(pov, resident, tf_, params_, band_rows=8)
    rec.append(((time.perf_counter() - t0) * 1e3, tiles.render_tiles.last_stats["kernel_ms"]))
    return fr


runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
for mode in ("off", "linear"):
    rec.clear()
    for key in T:
        T[key].clear()
    t, _, agg = runtime.replay(povs[3:23], man, cache, tf, params, prefetch=mode, keep_frames=False, render_fn=draw)
    r = np.array(rec)
    print(mode, {k: round(v, 3) if isinstance(v, float) else v for k, v in agg.items()},
          "draw wall %.3f ms, kernel %.3f ms" % tuple(r.mean(axis=0)),
          {k: (len(v), round(float(np.mean(v)), 3) if v else None) for k, v in T.items()}, flush=True)
pr = cProfile.Profile()
pr.enable()
runtime.replay(povs[23:43], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
