"""K2 lane occupancy: per-ray sample counts of config-3 frames (debug
output), and for warp tiles of several shapes the fraction of lane-iterations
that do work (sum of a tile's counts / (32 x its longest ray)), plus what a
warp that refills finished lanes from a queue of T consecutive tiles would
reach.

    python tools/diag_lanes.py [--frames 0,7,25,50]"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_00184_b200 import render, runtime, synth  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", default="0,7,25,50")
ap.add_argument("--size", type=int, default=1024)
args = ap.parse_args()

man, blobs = synth.turbulence_store()
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=args.size, height=args.size, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
frames = [int(f) for f in args.frames.split(",")]
need = sorted({a for k in frames for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
torch.cuda.synchronize()
for k in frames:
    vis = render.select_visible(povs[k], man)
    out, info, dbg = render.render_part(povs[k], {a: res[a] for a in vis}, tf, params, debug=True)
    torch.cuda.synchronize()
    ns = dbg["nsamp"].cpu().numpy().astype(np.int64)
    H, W = ns.shape
    rec = {"frame": k, "samples": int(ns.sum()), "rays_nonzero": int((ns > 0).sum()), "max": int(ns.max())}
    for tw, th in ((4, 8), (8, 4), (2, 16), (16, 2)):
        t = ns[: H // th * th, : W // tw * tw].reshape(H // th, th, W // tw, tw).transpose(0, 2, 1, 3)
        t = t.reshape(-1, tw * th)
        mx = t.max(axis=1)
        rec[f"eff_{tw}x{th}"] = round(float(t.sum() / max(1, 32 * mx.sum())), 4)
        # warp refilling from T tiles stacked vertically: lanes busy until the
        # queue's work runs out; bound = total / (32 * max(ceil-ish drain))
        for T in (2, 4, 8):
            g = t[: (len(t) // T) * T]
            # tiles are in row-major order over (tile row, tile col); group T
            # tiles of the same column, consecutive tile rows
            nty, ntx = H // th, W // tw
            tt = t.reshape(nty, ntx, 32)[: nty // T * T].reshape(nty // T, T, ntx, 32).transpose(0, 2, 1, 3)
            tt = tt.reshape(-1, T * 32)
            work = tt.sum(axis=1)
            # greedy list scheduling of the queue's rays onto 32 lanes in order
            import heapq
            busy = 0
            for row in tt[:: max(1, len(tt) // 2000)]:
                lanes = [0] * 32
                for r in row:
                    heapq.heapreplace(lanes, lanes[0] + int(r))
                busy += max(lanes)
            sub = tt[:: max(1, len(tt) // 2000)].sum()
            rec[f"refill_{tw}x{th}_T{T}"] = round(float(sub / max(1, 32 * busy)), 4)
        del g
    print(json.dumps(rec), flush=True)
