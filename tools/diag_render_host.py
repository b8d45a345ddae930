"""Break down render_part's host wall time (no replay, blocks resident)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import _lib, render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
need = sorted({a for k in range(3, 23) for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
torch.cuda.synchronize()
lib = _lib.lib()
orig = lib.afam_render
T = {"c_call": [], "sync": []}


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
    T["sync"].append((time.perf_counter() - t0) * 1e3)


torch.cuda.Stream.synchronize = sync
for host_out in (False, True):
    for key in T:
        T[key].clear()
    walls, kms = [], []
    for k in range(3, 23):
        blocks = {a: res[a] for a in render.select_visible(povs[k], man)}
        t0 = time.perf_counter()
        out, info, _ = render.render_part(povs[k], blocks, tf, params, host_out=host_out)
        walls.append((time.perf_counter() - t0) * 1e3)
        kms.append(info["kernel_ms"])
    print(f"host_out={host_out}: wall {np.mean(walls[2:]):.3f} ms, kernel {np.mean(kms[2:]):.3f} ms, "
          f"afam_render call {np.mean(T['c_call'][2:]):.3f} ms, sync {np.mean(T['sync'][2:]):.3f} ms", flush=True)
