"""Out-of-core replay from a store on disk vs from pinned host memory:
config-4 orbit (ModelCache(200), linear prefetch) over the blocks the first
`--frames` poses touch, written to a temporary store directory."""
import argparse
import json
import sys
import tempfile
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, store, tiles  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=40)
args = ap.parse_args()
man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)[: args.frames + 3]
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
need = sorted({a for p in runtime.orbit_trajectory(100, radius=2.0) for a in render.select_visible(p, man)})
root = tempfile.mkdtemp(prefix="afam_store_")
t0 = time.perf_counter()
sub = type(man)(levels=man.levels, micro_dims=man.micro_dims, finest_blocks_per_axis=man.finest_blocks_per_axis,
                volume_dims=man.volume_dims, bounds=man.bounds, degree=man.degree)
for a in man.entries:
    sub.entries[a] = man.entries[a]
store.write_store(root, sub, {a: bytes(blobs[a]) for a in need})
wr = time.perf_counter() - t0
for kind in ("memory", "files"):
    ds = DeviceStore(201, 65)
    src = (lambda a: blobs[a]) if kind == "memory" else None
    cache = runtime.ModelCache(200, runtime.make_loader(root, sub, ds, source=src))
    samples = [0]

    def draw(pov, resident, tf_, params_):
        fr = tiles.render_tiles(pov, resident, tf_, params_, band_rows=8)
        samples[0] += tiles.render_tiles.last_stats["samples"]
        return fr

    class Counted:  # split at the GPU wait, as bench.py's e2e draw (prefetch while the GPU marches)
        def __init__(self, pending):
            self.pending = pending

        def done(self):
            return self.pending.done()

        def result(self):
            fr = self.pending.result()
            samples[0] += tiles.render_tiles.last_stats["samples"]
            return fr

    draw.submit = lambda pov, resident, tf_, params_: Counted(
        tiles.submit_tiles(pov, resident, tf_, params_, band_rows=8))

    runtime.replay(povs[:3], sub, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
    samples[0] = 0
    c0 = cache.counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, agg = runtime.replay(povs[3:], sub, cache, tf, params, prefetch="linear", keep_frames=False,
                               render_fn=draw)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    c1 = cache.counters()
    print(json.dumps({"source": kind, "frames": len(povs) - 3, "samples_per_s": samples[0] / el,
                      "mean_caching_ms": agg["mean_caching_ms"], "mean_rendering_ms": agg["mean_rendering_ms"],
                      "miss_rate": agg["miss_rate"], "bytes_loaded": c1["bytes_loaded"] - c0["bytes_loaded"],
                      "store_blocks": len(need), "store_write_s": wr}), flush=True)
