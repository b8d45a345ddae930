"""K2 on the config-3 geometry at p = 2 and p = 3 ("Degree 3
(state it; also report p=2)"): the same synthetic turbulence field fitted at
each degree, frames 3..22 of the orbit with the visible blocks resident,
device time per 1024^2 frame (CUDA events on the render stream)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_00184_b200 import render, runtime, synth  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

povs = runtime.orbit_trajectory(100, radius=2.0)
params = render.RenderParams(width=1024, height=1024, sample_distance=1e-3)
tf = render.TransferFunction.ml_preset()
degrees = [int(v) for v in sys.argv[1:]] or [2, 3]
for degree in degrees:
    man, blobs = synth.turbulence_store(degree=degree)
    need = sorted({a for k in range(3, 23) for a in render.select_visible(povs[k], man)})
    ds = DeviceStore(len(need) + 1, 65)
    res = {a: ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in need}
    frames = [{a: res[a] for a in render.select_visible(povs[k], man)} for k in range(3, 23)]
    for k in range(3):
        render.render(povs[3 + k], frames[k], tf, params)
    torch.cuda.synchronize()
    ms, samples, shaded = [], 0, 0
    for k in range(20):
        render.render(povs[3 + k], frames[k], tf, params)
        st = render.render.last_stats
        ms.append(st["kernel_ms"])
        samples += st["samples"]
        shaded += st["shaded_samples"]
    print(json.dumps({"degree": degree, "frames": "3..22", "kernel_ms_mean": float(np.mean(ms)),
                      "samples_per_frame": samples / 20, "samples_per_s": samples / (sum(ms) * 1e-3),
                      "shaded_frac": shaded / samples, "fp64_slots": int(sum(1 for b in res.values()
                                                                             if getattr(b, "fp64", False)))}),
          flush=True)
    del res, frames, ds
