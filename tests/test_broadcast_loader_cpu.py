"""Shared cache misses across ranks (tiles.BroadcastLoader) on
CPU: gloo, world size 2 and 3, CPU staging tensors and a host stand-in for
the device store.  Checks the lockstep protocol the GPU path relies on:

* every miss is read from the host by exactly one rank (rank i % N for the
  i-th miss) and every other rank receives the same bytes;
* ranks whose local "rendering done" answers differ still prefetch the same
  blocks (LockstepDone: rank 0 decides), so their caches stay identical;
* a corrupt image raises the same exception class on every rank.
"""

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class HostStore:
    """Stand-in for DeviceStore: slots hold the bytes put_mfa_device copied."""

    def __init__(self, slots, max_ncp):
        self.device = -1
        self.max_ncp = max_ncp
        self.free = list(range(slots - 1, -1, -1))
        self.data = {}

    def alloc(self):
        return self.free.pop()

    def release(self, slot):
        self.data.pop(slot, None)
        self.free.append(slot)

    def put_mfa_device(self, slot, dptr, nbytes, degree, ncp, extent, stream=None):
        self.data[slot] = (C.string_at(dptr, nbytes), degree, ncp)


class Flaky:
    """A rendering_done whose answer differs per rank (only rank 0's counts)."""

    def __init__(self, rank, after):
        self.rank, self.calls, self.after = rank, 0, after

    def is_set(self):
        self.calls += 1
        return self.calls > self.after if self.rank == 0 else (self.calls % 2 == 0)


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2409_00184_b200 import runtime, synth, tiles
    from paper_2409_00184_b200.errors import FormatError

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    man, blobs = synth.field_store(levels=2, coarsest=2, micro=5, degree=2, ncp_of=lambda a: 4)
    addrs = sorted(blobs)
    bad = addrs[-1]
    src = dict(blobs)
    src[bad] = bytes(blobs[bad])[:-4]  # truncated: FormatError on the reading rank
    store = HostStore(len(addrs) + 1, 4)
    loader = tiles.BroadcastLoader(man, store, lambda a: src[a], device="cpu")
    cache = runtime.ModelCache(6, loader)
    log = []
    # frame misses (deterministic), then a lockstep prefetch that rank 0 stops after 3 loads
    cache.begin_frame(addrs[:4])
    cache.fetch_many(addrs[:4])
    done = loader.lockstep(Flaky(rank, after=3))
    n = 0
    for a in addrs[4:-1]:
        if a in cache:
            continue
        if done.is_set():
            break
        cache.fetch(a, record=False)
        n += 1
    log.append(("prefetched", n))
    try:
        cache.fetch(bad)
        log.append(("bad", "no error"))
    except FormatError:
        log.append(("bad", "FormatError"))
    res = [(a.key, store.data[b.slot][0] == bytes(blobs[a])) for a, b in zip(cache.resident_addresses(),
                                                                          [cache.fetch(x, record=False) for x in
                                                                           cache.resident_addresses()])]
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as fh:
        fh.write(repr({"log": log, "resident": res, "h2d": loader.h2d_bytes, "recv": loader.recv_bytes,
                       "misses": loader.misses}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_broadcast_loader_lockstep(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    out = [eval((tmp_path / f"r{r}.txt").read_text()) for r in range(world)]
    # identical cache contents and decisions on every rank; bytes intact
    for o in out[1:]:
        assert o["resident"] == out[0]["resident"]
        assert o["log"] == out[0]["log"]
        assert o["misses"] == out[0]["misses"]
    assert all(ok for _, ok in out[0]["resident"])
    assert out[0]["log"][0] == ("prefetched", 3)  # rank 0's answer governs every rank
    assert out[0]["log"][1] == ("bad", "FormatError")
    # every image crossed the host link once: what one rank read, the others received
    total_h2d = sum(o["h2d"] for o in out)
    for o in out:
        assert o["h2d"] + o["recv"] == total_h2d
    assert sum(1 for o in out if o["h2d"] > 0) == world  # misses rotate over the ranks
