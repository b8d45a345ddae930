"""Phases of render.png_bytes_gpu on a 1024^2 frame: H2D, afam_png_deflate
(kernels + host Huffman build), D2H, host CRC/chunking."""
import ctypes as C
import sys
import time
import zlib

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_00184_b200 import _lib  # noqa: E402

rng = np.random.default_rng(0)
H = W = 1024
yy, xx = np.mgrid[0:H, 0:W]
img = np.zeros((H, W, 4), np.uint8)
img[..., 0] = (xx * 255 // W).astype(np.uint8)
img[..., 1] = (yy * 255 // H).astype(np.uint8)
img[..., 2] = (rng.random((H, W)) * 40).astype(np.uint8)
img[..., 3] = 255
for rep in range(4):
    t0 = time.perf_counter()
    d = torch.from_numpy(img).cuda()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    cap = int(((4 * W + 1) * 15 // 8 + 16) * H + 2048)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb, ad = C.c_uint64(), C.c_uint32()
    _lib.check(_lib.lib().afam_png_deflate(C.c_void_p(d.data_ptr()), W, H, C.c_void_p(out.data_ptr()), cap,
                                           C.byref(nb), C.byref(ad), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    body = out[: nb.value].cpu().numpy().tobytes()
    t3 = time.perf_counter()
    zlib.crc32(body)
    t4 = time.perf_counter()
    print("h2d %.2f deflate %.2f d2h %.2f crc %.2f ms  (%d bytes)" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3,
                                                                     (t4 - t3) * 1e3, nb.value))
