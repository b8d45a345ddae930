"""render_part inside the replay loop, with checkpoints (host wall per phase)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import _lib, render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore, as_device_blocks  # noqa: E402

man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
ds = DeviceStore(201, 65)
cache = runtime.ModelCache(200, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
P = []


def draw(pov, blocks, tf_, params_):
    t = [time.perf_counter()]
    addrs = sorted(blocks)
    store, slots = as_device_blocks([blocks[a] for a in addrs], 0)
    H, W = 1024, 1024
    fr = render._frame_struct(pov, tf_, params_, H, 1, 0, False)
    out = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
    stats = torch.empty(6, dtype=torch.int64, device="cuda")
    sl = np.ascontiguousarray(slots, dtype=np.int32)
    s_obj = torch.cuda.current_stream()
    ez = torch.cuda.Event(enable_timing=True)
    ez.record(s_obj)
    t.append(time.perf_counter())
    _lib.check(_lib.lib().afam_render(store.handle, C.byref(fr), sl.ctypes.data_as(C.c_void_p), len(sl),
                                      C.c_void_p(out.data_ptr()), C.c_void_p(stats.data_ptr()), None, None,
                                      C.c_void_p(int(s_obj.cuda_stream))))
    t.append(time.perf_counter())
    stage = render._pinned_stage(H * W * 4)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_obj)
    stage[:48].view(torch.int64).copy_(stats, non_blocking=True)
    stage[64:64 + H * W * 4].view(H, W, 4).copy_(out, non_blocking=True)
    e1.record(s_obj)
    t.append(time.perf_counter())
    s_obj.synchronize()
    t.append(time.perf_counter())
    o = stage[64:64 + H * W * 4].view(H, W, 4).clone()
    t.append(time.perf_counter())
    f = render.Frame(W, H, o.numpy())
    t.append(time.perf_counter())
    kms = C.c_float()
    _lib.check(_lib.lib().afam_render_elapsed(store.handle, C.byref(kms)))
    P.append([(b - a) * 1e3 for a, b in zip(t[:-1], t[1:])] + [kms.value, e0.elapsed_time(e1), ez.elapsed_time(e0)])
    return f


runtime.replay(povs[:3], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
print("stream", torch.cuda.current_stream(), torch.cuda.current_stream().cuda_stream)
x = torch.empty(64 << 20, dtype=torch.uint8, device="cuda"); h = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); h.copy_(x, non_blocking=True); b.record(); torch.cuda.synchronize()
    print("D2H 64 MiB pinned: %.1f GB/s" % (64 * 2**20 / a.elapsed_time(b) / 1e6))
for mode in ("off", "linear", "off", "off"):
    P.clear()
    t, _, agg = runtime.replay(povs[3:23], man, cache, tf, params, prefetch=mode, keep_frames=False, render_fn=draw)
    print(mode, {k: round(v, 3) if isinstance(v, float) else v for k, v in agg.items()})
    print("   prep %.3f | afam_render %.3f | d2h enqueue %.3f | sync %.3f | clone %.3f | Frame %.3f | kernel %.3f | d2h dev %.3f | gpu start->d2h %.3f"
          % tuple(np.mean(P, axis=0)), flush=True)
