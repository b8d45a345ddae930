"""Host-side time per frame of the pipelined replay (config-4 orbit): the
prefetch loop, the next frame's caching, the launch (submit) and the wait
in result(), to see whether the GPU or the host paces the loop.

    python tools/diag_hostpath.py [frames]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, tiles  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 97
man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
acc = {"prefetch": 0.0, "caching": 0.0, "submit": 0.0, "result": 0.0, "loads_host": 0.0}
orig_prefetch, orig_cache = runtime.prefetch_loop, runtime.cache_frame


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t
    return w


runtime.prefetch_loop = timed("prefetch", orig_prefetch)
runtime.cache_frame = timed("caching", orig_cache)


class P:
    def __init__(self, p):
        self.p = p

    def done(self):
        return self.p.done()

    def result(self):
        t = time.perf_counter()
        r = self.p.result()
        acc["result"] += time.perf_counter() - t
        return r


def draw(pov, resident, tf_, params_):
    return tiles.render_tiles(pov, resident, tf_, params_, band_rows=8)


def submit(pov, resident, tf_, params_):
    t = time.perf_counter()
    p = tiles.submit_tiles(pov, resident, tf_, params_, band_rows=8)
    acc["submit"] += time.perf_counter() - t
    return P(p)


draw.submit, draw.frames_in_flight = submit, 2
ds = DeviceStore(201, 65)
loader = runtime.make_loader(None, man, ds, source=lambda a: blobs[a])
orig_loader = loader.__call__


class L:  # time spent in the loader (host side of each load)
    def __init__(self, inner):
        self.inner = inner
        self.release = inner.release
        self.sync = inner.sync

    def __call__(self, a):
        t = time.perf_counter()
        try:
            return self.inner(a)
        finally:
            acc["loads_host"] += time.perf_counter() - t


cache = runtime.ModelCache(200, L(loader))
runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
torch.cuda.synchronize()
for k in acc:
    acc[k] = 0.0
t0 = time.perf_counter()
tim, _, _ = runtime.replay(povs[3:3 + nfr], man, cache, tf, params, prefetch="linear", keep_frames=False,
                           render_fn=draw)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(json.dumps({"ms_per_frame": 1e3 * el / nfr, **{k + "_ms": 1e3 * v / nfr for k, v in acc.items()},
                  "loaded": sum(t.prefetch_models_loaded for t in tim)}))
