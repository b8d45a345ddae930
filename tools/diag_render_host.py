"""Where the host time of render.render() goes on resident config-3 blocks:
total call vs kernel_ms, and the cost of materialising the 4 MB frame."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
need = sorted({a for k in range(3, 23) for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
frames = [{a: res[a] for a in render.select_visible(povs[k], man)} for k in range(3, 23)]
for k in range(3):
    render.render(povs[3 + k], frames[k], tf, params)
torch.cuda.synchronize()
tot, kern = [], []
for k in range(20):
    t0 = time.perf_counter()
    fr = render.render(povs[3 + k], frames[k], tf, params)
    tot.append((time.perf_counter() - t0) * 1e3)
    kern.append(render.render.last_stats["kernel_ms"])
print("render() %.3f ms, kernel %.3f ms" % (np.median(tot), np.median(kern)))
src = torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True)
for name, fn in (("clone pinned->torch", lambda: src.clone()),
                 ("np.empty+copyto", lambda: np.copyto(np.empty(4 << 20, np.uint8), src.numpy())),
                 ("np.array copy", lambda: np.array(src.numpy()))):
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        x = fn()
        ts.append((time.perf_counter() - t0) * 1e3)
        del x
    print("%s %.3f ms" % (name, np.median(ts)))
