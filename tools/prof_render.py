"""Profiling driver: render config-3 frames (blocks of the frame resident in HBM).

    python tools/prof_render.py [--frames 7,8] [--warm 1] [--size 1024]

Used under ncu (launch list / --set full capture of render_kernel)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2409_00184_b200 import render, runtime, synth  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", default="7")
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--flush", action="store_true")
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
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for k in frames[:1] * args.warm + frames:
    vis = render.select_visible(povs[k], man)
    if args.flush:
        flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, info, _ = render.render_part(povs[k], {a: res[a] for a in vis}, tf, params)
    torch.cuda.synchronize()
    print(f"frame {k}: {info['samples']} samples, {len(vis)} blocks, {1e3 * (time.perf_counter() - t0):.2f} ms wall",
          flush=True)
