"""Shared cache misses on the GPU (tiles.BroadcastLoader): two processes
(gloo carries the broadcasts; both share the test box's one GPU -- on a node
each rank has its own GPU and NCCL moves the images over NVLink) replay an
orbit through ModelCache + linear prefetch, every miss read from the host by
one rank and realigned from the received device copy by the others
(afam_store_put_mfa_device).  Every frame must equal the single-process
replay's byte for byte, and the two ranks' caches must hold the same blocks."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2409_00184_b200 import render, runtime, synth

    # 73 blocks over 3 LODs; the 8-14 visible blocks per frame and 40 over
    # the orbit make a 16-block cache evict
    man, blobs = synth.field_store(levels=3, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 6 + (a.lod % 2))
    povs = runtime.orbit_trajectory(8, radius=1.2)
    params = render.RenderParams(width=40, height=32, sample_distance=0.01)
    return man, blobs, povs, params, render.TransferFunction.ml_preset()


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2409_00184_b200 import runtime, tiles
    from paper_2409_00184_b200.device import DeviceStore

    man, blobs, povs, params, tf = _setup()
    cap = 16
    ds = DeviceStore(cap + 1, 9)
    loader = tiles.BroadcastLoader(man, ds, lambda a: blobs[a])
    cache = runtime.ModelCache(cap, loader)
    _, frames, agg = runtime.replay(povs, man, cache, tf, params, prefetch="linear")
    np.save(os.path.join(outdir, f"frames{rank}.npy"), np.stack([f.rgba for f in frames]))
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as fh:
        fh.write(repr({"resident": [a.key for a in cache.resident_addresses()], "h2d": loader.h2d_bytes,
                       "recv": loader.recv_bytes, "misses": loader.misses}))
    dist.barrier()
    dist.destroy_process_group()


def test_broadcast_loader_replay_matches_single_process(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    from paper_2409_00184_b200 import runtime
    from paper_2409_00184_b200.device import DeviceStore

    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    man, blobs, povs, params, tf = _setup()
    cap = 16
    ds = DeviceStore(cap + 1, 9)
    cache = runtime.ModelCache(cap, runtime.make_loader(None, man, ds, source=lambda a: blobs[a]))
    _, frames, _ = runtime.replay(povs, man, cache, tf, params, prefetch="off")
    want = np.stack([f.rgba for f in frames])
    r = [eval((tmp_path / f"r{k}.txt").read_text()) for k in range(2)]
    assert r[0]["resident"] == r[1]["resident"]
    assert r[0]["misses"] == r[1]["misses"] > 0
    assert r[0]["h2d"] > 0 and r[1]["h2d"] > 0  # misses rotate over the ranks
    assert r[0]["h2d"] + r[0]["recv"] == r[1]["h2d"] + r[1]["recv"]
    for k in range(2):
        np.testing.assert_array_equal(np.load(tmp_path / f"frames{k}.npy"), want)
