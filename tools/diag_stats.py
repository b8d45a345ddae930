"""K2 per-frame statistics on one config-3 frame: samples, shaded, exact-path
samples and exact owner evaluations (knext points) per sample."""
import sys
sys.path.insert(0, ".")
import bench
from paper_2409_00184_b200 import render, runtime
from paper_2409_00184_b200.device import DeviceStore
man, blobs, _ = bench.build_model(pinned=False)
povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
vis = render.select_visible(povs[5], man)
ds = DeviceStore(len(vis) + 1, 65)
res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
render.render(povs[5], res, tf, params)
st = render.render.last_stats
print({k: v for k, v in st.items()})
print("exact_cells per sample %.4f, exact samples per sample %.5f" % (st["exact_cells"] / st["samples"], st["exact_samples"] / st["samples"]))
