"""cProfile of the e2e replay loop (bench.run_e2e's path) on the host."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2409_00184_b200 import render, runtime  # noqa: E402

sys.argv = ["bench.py", "--e2e-steps", "40"]
args = bench.parse()
man, blobs, _ = bench.build_model(pinned=True)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
bench.run_e2e(args, man, blobs, povs, tf, params, 0, 1, 0)
pr = cProfile.Profile()
pr.enable()
r = bench.run_e2e(args, man, blobs, povs, tf, params, 0, 1, 0)
pr.disable()
print("value %.3e cach %.3f rend %.3f" % (r["value"], r["mean_caching_ms"], r["mean_rendering_ms"]))
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
