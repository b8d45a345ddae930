"""Frame egress: Frame.to_png_bytes on the GPU vs the reference's PIL/zlib
path, on 1024^2 config-3 frames."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
ks = [3, 40]
need = sorted({a for k in ks for a in render.select_visible(povs[k], man)})
ds = DeviceStore(len(need) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
for k in ks:
    fr = render.render(povs[k], {a: res[a] for a in render.select_visible(povs[k], man)}, tf, params)
    fr.to_png_bytes()  # warm-up
    t = time.perf_counter()
    for _ in range(10):
        g = fr.to_png_bytes()
    tg = (time.perf_counter() - t) / 10
    t = time.perf_counter()
    p = fr._to_png_bytes_pil()
    tp = time.perf_counter() - t
    print(json.dumps({"frame": k, "gpu_ms": tg * 1e3, "gpu_bytes": len(g), "pil_ms": tp * 1e3, "pil_bytes": len(p),
                      "raw_bytes": fr.rgba.nbytes}), flush=True)
