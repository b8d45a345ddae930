"""Small workloads for compute-sanitizer runs (tools/gpu_sanitize.sh).

    python tools/sanitize.py decode|render|eval|replay

decode  every K3 path (register-tiled, banded float32 / float64, tcgen05) on
        a few config-5 blocks (ncp 40..65, one ill-conditioned block)
render  K2 frames on a small two-LOD store (fast path, and the float64 path
        of an ill-conditioned block)
eval    K1 on a bucketed batch (n = 2^17: count / scan / scatter /
        unpermute) and on an unbucketed one
replay  ModelCache + linear prefetch on the frame thread while the GPU
        marches (cross-stream slot reuse, reader fences)
highdeg degree-5 blocks (the float64 any-degree path): K2 frames with a
        300-point transfer function, K3 decode (decode_any_kernel) next to
        degree-3 blocks, K1 points
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_00184_b200 import _lib, model, render, runtime, synth  # noqa: E402
from paper_2409_00184_b200.bspline import DECODE_PATHS, clamped_knots  # noqa: E402
from paper_2409_00184_b200.device import DeviceStore, stream_handle  # noqa: E402


def decode():
    man, blobs = synth.field_store(levels=1, coarsest=2, micro=65, degree=3, ncp_of=lambda a: 40 + 3 * sum(a.ijk))
    addrs = sorted(blobs)
    ds = DeviceStore(len(addrs) + 1, 65)
    slots = [ds.load_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod).slot for a in addrs]
    # an ill-conditioned (float64) block: ncp = m, endpoint-pinned fit of a rough field
    rng = np.random.default_rng(3)
    ctrl = (rng.standard_normal((65, 65, 65)) * 50).astype(np.float32)
    mm = model.MicroModel(3, np.stack([clamped_knots(65, 3)] * 3).astype(np.float32), ctrl,
                          man.entries[addrs[0]].extent, 1)
    slots.append(ds.load_model(mm).slot)
    sl = np.asarray(slots, dtype=np.int32)
    out = torch.empty(len(sl) * 65 ** 3, dtype=torch.float32, device="cuda")
    for path in ("auto", "cuda_cores", "tensor_cores"):
        ntc = C.c_int32(0)
        _lib.check(_lib.lib().afam_decode_grid_ex(ds.handle, sl.ctypes.data_as(C.c_void_p), len(sl), 65,
                                                  C.c_void_p(out.data_ptr()), DECODE_PATHS[path], C.byref(ntc),
                                                  C.c_void_p(stream_handle())))
    torch.cuda.synchronize()
    print("decode ok", len(sl), "blocks")


def render_frames():
    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 7)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    a0 = sorted(models)[-1]  # one ill-conditioned block (max |c| > 4: the float64 path)
    m0 = models[a0]
    models[a0] = model.MicroModel(3, m0.knots, m0.control * 40.0 - 20.0, m0.extent, m0.lod)
    tf = render.TransferFunction.ml_preset()
    params = render.RenderParams(width=24, height=20, sample_distance=0.01)
    for pos in ([0.2, 0.3, 1.9], [1.4, 1.1, 1.3]):
        p = np.asarray(pos)
        pov = render.PointOfView(p, -p, [0, 1, 0], 50.0)
        vis = render.select_visible(pov, man, params.aspect)
        render.render(pov, {a: models[a] for a in vis}, tf, params)
    torch.cuda.synchronize()
    print("render ok")


def eval_points():
    man, blobs = synth.field_store(levels=1, coarsest=2, micro=9, degree=3, ncp_of=lambda a: 7)
    addrs = sorted(blobs)
    ds = DeviceStore(len(addrs), 9)
    slots = np.array([ds.load_mfa(blobs[a], 7, man.entries[a].extent, a.lod).slot for a in addrs], np.int32)
    rng = np.random.default_rng(0)
    for n in (1 << 17, 1000):
        u = torch.from_numpy(rng.uniform(0, 1, size=(n, 3))).cuda()
        sl = torch.from_numpy(slots[rng.integers(0, len(slots), size=n)]).cuda()
        val = torch.empty(n, dtype=torch.float32, device="cuda")
        grad = torch.empty((n, 3), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().afam_eval_points(ds.handle, C.c_void_p(sl.data_ptr()), 0, C.c_void_p(u.data_ptr()), n,
                                               C.c_void_p(val.data_ptr()), C.c_void_p(grad.data_ptr()),
                                               _lib.AFAM_EVAL_PARAM, C.c_void_p(stream_handle())))
    torch.cuda.synchronize()
    print("eval ok")


def replay():
    man, blobs = synth.field_store(levels=3, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 6 + (a.lod % 2))
    povs = runtime.orbit_trajectory(6, radius=1.2)
    params = render.RenderParams(width=24, height=20, sample_distance=0.02)
    ds = DeviceStore(17, 9)
    cache = runtime.ModelCache(16, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
    runtime.replay(povs, man, cache, render.TransferFunction.ml_preset(), params, prefetch="linear",
                   keep_frames=False)  # render.render: two frames in flight, next caching overlapped
    torch.cuda.synchronize()
    print("replay ok")


def highdeg():
    from paper_2409_00184_b200 import bspline

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=5, ncp_of=lambda a: 7)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    rng = np.random.default_rng(1)
    cp = np.column_stack([np.sort(rng.uniform(0, 1, 300)), rng.uniform(0, 1, (300, 3))])
    op = np.column_stack([np.sort(rng.uniform(0, 1, 90)), rng.uniform(0, 0.1, 90)])
    tf = render.TransferFunction(cp, op)
    params = render.RenderParams(width=24, height=20, sample_distance=0.01)
    pov = render.PointOfView([0.2, 0.3, 1.9], [-0.2, -0.3, -1.9], [0, 1, 0], 50.0)
    vis = render.select_visible(pov, man, params.aspect)
    render.render(pov, {a: models[a] for a in vis}, tf, params)
    m5 = models[vis[0]]
    ds = DeviceStore(2, 9)
    ds.put_model(0, m5)
    c3 = rng.normal(size=(9, 9, 9)).astype(np.float32)
    ds.put_model(1, model.MicroModel(3, np.stack([clamped_knots(9, 3)] * 3).astype(np.float32), c3,
                                     np.array([[0, 1.0]] * 3), 1))
    bspline.decode_slots(ds, [0, 1], 17)
    bspline.evaluate_points_with_gradient(m5.control, 5, rng.uniform(0, 1, (1000, 3)), knots=tuple(m5.knots))
    torch.cuda.synchronize()
    print("highdeg ok")


if __name__ == "__main__":
    {"decode": decode, "render": render_frames, "eval": eval_points, "replay": replay, "highdeg": highdeg}[sys.argv[1]]()
