"""A/B of runtime.replay's frame schedule on the config-4 workload (e2e leg
of bench.py): AFAM_REPLAY_OVERLAP=1 (next frame's caching while the GPU
renders) vs 0 (the reference's strict order), alternated.

    python tools/diag_replay.py [frames] [rounds]
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime, tiles  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()


def draw(pov, resident, tf_, params_):
    return tiles.render_tiles(pov, resident, tf_, params_, band_rows=8)


class Timed:  # collects each frame's kernel time and its stream time (incl. waits for its uploads)
    def __init__(self, p, ea, eb):
        self.p, self.ea, self.eb = p, ea, eb

    def done(self):
        return self.p.done()

    def result(self):
        f = self.p.result()
        kms.append(tiles.render_tiles.last_stats["kernel_ms"])
        spans.append((self.ea, self.eb))
        return f


kms, spans = [], []


def _submit(pov, resident, tf_, params_):
    st = render._render_stream(torch.device("cuda", 0))
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(st)
    p = tiles.submit_tiles(pov, resident, tf_, params_, band_rows=8)
    eb.record(st)
    return Timed(p, ea, eb)


draw.submit = _submit
draw.frames_in_flight = 2
for r in range(rounds):
    for mode in os.environ.get("MODES", "2,1,0").split(","):  # depth 2, depth 1 (overlapped caching), strict order
        os.environ["AFAM_REPLAY_OVERLAP"] = "0" if mode == "0" else "1"
        os.environ["AFAM_REPLAY_DEPTH"] = "2" if mode == "2" else "1"
        ds = DeviceStore(201, 65)
        cache = runtime.ModelCache(200, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
        runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
        torch.cuda.synchronize()
        kms.clear()
        spans.clear()
        t0 = time.perf_counter()
        tim, _, agg = runtime.replay(povs[3:3 + nfr], man, cache, tf, params, prefetch="linear",
                                     keep_frames=False, render_fn=draw)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        print(json.dumps({"overlap": mode, "frames": nfr, "ms_per_frame": 1e3 * el / nfr,
                          "caching_ms": sum(t.caching_ms for t in tim) / nfr,
                          "rendering_ms": sum(t.rendering_ms for t in tim) / nfr,
                          "loaded": sum(t.prefetch_models_loaded for t in tim),
                          "kernel_ms": sum(kms) / max(1, len(kms)),
                          # stream time per frame (pack upload + waits for its uploads + kernels) and the
                          # GPU gap between a frame's end and the next frame's start on the render stream
                          "stream_ms": sum(a.elapsed_time(b) for a, b in spans) / max(1, len(spans)),
                          "gap_ms": sum(spans[j][1].elapsed_time(spans[j + 1][0]) for j in range(len(spans) - 1))
                          / max(1, len(spans) - 1)}), flush=True)
        del cache, ds
