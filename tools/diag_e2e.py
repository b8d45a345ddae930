"""e2e replay variants: where the wall time per frame goes beyond the kernel
(GIL switch interval, prefetch thread, per-frame thread start)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402

variant = sys.argv[1:] or ["base"]
sys.argv = ["bench.py", "--e2e-steps", "40"]
args = bench.parse()
man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
for v in variant:
    if v == "si":
        sys.setswitchinterval(2e-4)
    if v == "nopf":
        runtime.PREDICTORS["linear"] = None
    r = bench.run_e2e(args, man, blobs, povs, tf, params, 0, 1, 0)
    n = r["steps"]
    print(v, "value %.3e  cach %.3f  rend %.3f  wall/frame %.3f ms" % (
        r["value"], r["mean_caching_ms"], r["mean_rendering_ms"], 1.267e8 / r["value"] * 1e3))
