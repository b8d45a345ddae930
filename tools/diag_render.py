"""Diagnostic: render_part timing with/without L2 flush, big vs small store."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2409_00184_b200 import render, runtime, synth
from paper_2409_00184_b200.device import DeviceStore

man, blobs = synth.turbulence_store()
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
big = DeviceStore(len(blobs) + 1, 65)
res_big = {a: big.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

def timeit(res, k, do_flush):
    pov = povs[k]
    vis = render.select_visible(pov, man)
    blocks = {a: res[a] for a in vis}
    if do_flush:
        flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    out, info, _ = render.render_part(pov, blocks, tf, params)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3, info["samples"]

for k in range(3, 8):
    print("big noflush", k, timeit(res_big, k, False), flush=True)
for k in range(3, 8):
    print("big flush", k, timeit(res_big, k, True), flush=True)
small = DeviceStore(201, 65)
for k in range(3, 8):
    vis = render.select_visible(povs[k], man)
    res_small = {a: small.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
    torch.cuda.synchronize()
    print("small noflush", k, timeit(res_small, k, False), flush=True)
    print("small flush", k, timeit(res_small, k, True), flush=True)
    for b in res_small.values():
        small.release(b.slot)
