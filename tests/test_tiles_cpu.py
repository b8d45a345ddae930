"""Multi-process (gloo, world_size 2) tests of the image-band partitioning and
the rank-0 gather (the host side of the multi-GPU path; CPU tensors)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_00184_b200 import tiles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_part_rows_cover_frame_once():
    for H in (1, 7, 64, 1000, 1024):
        for br in (1, 8, 16):
            for n in (1, 2, 3, 8):
                allr = np.concatenate([tiles.part_rows(H, br, n, p) for p in range(n)])
                assert sorted(allr.tolist()) == list(range(H))


def test_part_rows_match_library():
    from paper_2409_00184_b200 import _lib

    for H, br, n in [(1024, 8, 8), (50, 4, 3), (7, 16, 2)]:
        for p in range(n):
            assert len(tiles.part_rows(H, br, n, p)) == _lib.lib().afam_frame_rows(H, br, n, p)


def test_assemble_inverts_partition():
    H, W, br, n = 37, 5, 4, 3
    frame = torch.arange(H * W * 4, dtype=torch.int32).reshape(H, W, 4)
    parts = [frame[torch.as_tensor(tiles.part_rows(H, br, n, p))] for p in range(n)]
    assert torch.equal(tiles.assemble(parts, H, br), frame)


def _worker(rank, world, port, H, W, br, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2409_00184_b200 import tiles as t

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    frame = torch.arange(H * W * 4, dtype=torch.int32).reshape(H, W, 4)
    mine = frame[torch.as_tensor(t.part_rows(H, br, world, rank))]
    full = t.gather_bands(mine, H, br)
    ok = bool(torch.equal(full, frame)) if rank == 0 else full is None
    with open(os.path.join(outdir, f"r{rank}"), "w") as fh:
        fh.write("1" if ok else "0")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_bands_gloo(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), 50, 6, 8, str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"r{r}").read_text() == "1" for r in range(world))


def _shard_worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2409_00184_b200 import tiles as t
    from paper_2409_00184_b200.partition import BlockAddress

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    # the config-3 skeleton's addresses, in a scrambled order on every rank
    addrs = [BlockAddress(l, (i, j, k)) for l, b in ((1, 16), (2, 8), (3, 4), (4, 2))
             for i in range(b) for j in range(b) for k in range(b)]
    rng = np.random.default_rng(rank)
    mine = t.shard_blocks([addrs[i] for i in rng.permutation(len(addrs))])  # rank/world from the process group
    got = [None] * world
    dist.all_gather_object(got, [(a.lod, *a.ijk) for a in mine])
    ok = True
    if rank == 0:
        flat = [x for part in got for x in part]
        ok = sorted(flat) == sorted((a.lod, *a.ijk) for a in addrs) and len(set(flat)) == len(flat)
        ok = ok and max(map(len, got)) - min(map(len, got)) <= 1
    with open(os.path.join(outdir, f"s{rank}"), "w") as fh:
        fh.write("1" if ok else "0")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_blocks_gloo(world, tmp_path):
    """Grid-decode sharding (config 5): every block on exactly
    one rank, balanced, the same split whatever order each rank lists them in."""
    mp.spawn(_shard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"s{r}").read_text() == "1" for r in range(world))
