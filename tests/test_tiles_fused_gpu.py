"""The fused band gather (tiles.render_tiles_fused): two processes (gloo for
the handle exchange and the barrier) render their interleaved bands straight
into rank 0's frame buffer through CUDA IPC (AFAM_RENDER_FULL_FRAME).  Both
processes share the one GPU of the test box; on a node every rank has its
own GPU and the stores go over NVLink.  The frame must equal a single-GPU
render byte for byte."""

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


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2409_00184_b200 import model, render, synth, tiles

    man, blobs = synth.field_store(levels=2, coarsest=1, micro=9, degree=3, ncp_of=lambda a: 7)
    models = {a: model.deserialize(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    pov = render.PointOfView([0.2, 0.3, 1.9], [-0.1, -0.15, -1.0], [0, 1, 0], 50.0)
    params = render.RenderParams(width=48, height=40, sample_distance=0.01)
    tf = render.TransferFunction.ml_preset()
    vis = render.select_visible(pov, man, params.aspect)
    peer = tiles.PeerFrame(params.height, params.width)
    fr = tiles.render_tiles_fused(pov, {a: models[a] for a in vis}, tf, params, peer, band_rows=4)
    if rank == 0:
        np.save(os.path.join(outdir, "fused.npy"), fr.rgba)
        np.save(os.path.join(outdir, "single.npy"), render.render(pov, {a: models[a] for a in vis}, tf, params).rgba)
    dist.barrier()
    peer.close()
    dist.destroy_process_group()


def test_fused_band_gather_matches_single_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    fused = np.load(tmp_path / "fused.npy")
    single = np.load(tmp_path / "single.npy")
    assert fused.shape == single.shape
    np.testing.assert_array_equal(fused, single)
