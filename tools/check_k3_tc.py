"""K3 tensor-core decode check: all 4,680 config-3 blocks decoded onto 65^3,
a sample of blocks against the float64 oracle (1e-5 x range), and timing."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2409_00184_b200 import model  # noqa: E402
from paper_2409_00184_b200.bspline import decode_slots  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore  # noqa: E402

man, blobs, _ = bench.build_model(pinned=False)
addrs = sorted(blobs)
ds = DeviceStore(len(addrs) + 1, 65)
blocks = [ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in addrs]
torch.cuda.synchronize()
slots = [b.slot for b in blocks]
t0 = time.perf_counter()
got = decode_slots(ds, slots[:200], 65)
print("decode_slots(200) wall %.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
rng = np.random.default_rng(0)
worst = 0.0
for b in rng.choice(200, 24, replace=False):
    a = addrs[b]
    m = model.deserialize(bytes(blobs[a]), man.entries[a].ncp, man.entries[a].extent, a.lod)
    want = oracle.decode_grid(m.control, m.degree, 65)
    err = float(np.abs(got[b] - want).max())
    worst = max(worst, err)
    if err > 1e-5:
        idx = np.unravel_index(np.argmax(np.abs(got[b] - want)), want.shape)
        print("block", b, "ncp", m.control.shape[0], "err", err, "at", idx, got[b][idx], want[idx], flush=True)
print("TC=%s max |err| over 24 blocks: %.3e" % (os.environ.get("AFAM_DECODE_TC", "1"), worst), flush=True)
