"""Kernel microbenchmarks on the config-3 model (all 4,680 blocks resident):

  K3  decode_grid((65,65,65)) of every block  (BASELINE config 5)
  K1  2^24 random parameter points, incoherent (uniform slots) and coherent
      (slot-sorted), value-only and value+gradient

Prints one JSON line per measurement with the HBM roofline (algorithmic
bytes: K3 4*ncp^3 + 4*m^3 per block; K1 4*q^3 + 24 + 4 (+12) per sample).
"""
import ctypes as C
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00184_b200 import _lib  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

HBM = 6552.0
DEGREE = int(sys.argv[1]) if len(sys.argv) > 1 else 3  # the config-3 model fitted at this degree
if DEGREE == 3:
    man, blobs, _ = bench.build_model(pinned=False)
else:
    from paper_2409_00184_b200 import synth

    man, blobs = synth.turbulence_store(degree=DEGREE)
addrs = sorted(blobs)
ds = DeviceStore(len(addrs) + 1, 65)
blocks = [ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in addrs]
torch.cuda.synchronize()
lib = _lib.lib()
st = torch.cuda.current_stream()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        ev0.record(st)
        fn()
        ev1.record(st)
        torch.cuda.synchronize()
        best = min(best, ev0.elapsed_time(ev1))
    return best


# ---------------------------------------------------------------- K3
m = 65
slots = np.array([b.slot for b in blocks], dtype=np.int32)
ncps = np.array([b.ncp for b in blocks], dtype=np.int64)
out = torch.empty(len(slots) * m ** 3, dtype=torch.float32, device="cuda")


def k3():
    _lib.check(lib.afam_decode_grid(ds.handle, slots.ctypes.data_as(C.c_void_p), len(slots), m,
                                    C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))


ms = timed(k3, 3)
nbytes = float((4 * ncps ** 3).sum() + 4 * m ** 3 * len(slots))
print(json.dumps({"kernel": "K3 decode_grid", "degree": DEGREE, "blocks": len(slots), "m": m, "ms": ms,
                  "samples_per_s": len(slots) * m ** 3 / (ms * 1e-3), "hbm_gbs": nbytes / (ms * 1e-3) / 1e9,
                  "frac_of_hbm": nbytes / (ms * 1e-3) / 1e9 / HBM}), flush=True)

# ---------------------------------------------------------------- K1
n = 1 << 24
rng = np.random.default_rng(0)
u = torch.from_numpy(rng.uniform(0, 1, size=(n, 3))).cuda()
sl_rand = torch.from_numpy(rng.integers(0, len(slots), size=n).astype(np.int32)).cuda()
sl_rand = torch.from_numpy(slots).cuda()[sl_rand.long()].int()
sl_sorted = torch.sort(sl_rand).values.contiguous()
val = torch.empty(n, dtype=torch.float32, device="cuda")
grad = torch.empty((n, 3), dtype=torch.float32, device="cuda")
mean_q3 = (DEGREE + 1) ** 3
for name, sl in (("incoherent", sl_rand), ("coherent", sl_sorted)):
    for g in (False, True):
        def k1():
            _lib.check(lib.afam_eval_points(ds.handle, C.c_void_p(sl.data_ptr()), 0, C.c_void_p(u.data_ptr()), n,
                                            C.c_void_p(val.data_ptr()), C.c_void_p(grad.data_ptr()) if g else None,
                                            _lib.AFAM_EVAL_PARAM, C.c_void_p(st.cuda_stream)))
        ms = timed(k1)
        per = 4 * mean_q3 + 24 + 4 + 4 + (12 if g else 0)
        print(json.dumps({"kernel": "K1 eval_points", "degree": DEGREE, "batch": name, "gradient": g, "n": n, "ms": ms,
                          "samples_per_s": n / (ms * 1e-3), "alg_bytes_per_sample": per,
                          "hbm_gbs": n * per / (ms * 1e-3) / 1e9}), flush=True)
