"""Image-band parallel rendering over the GPUs of one node.

Each rank renders the frame's row bands b with b % world == rank (8-row
bands by default, interleaved for load balance: early termination and cube
coverage vary across the image) into one packed buffer; one collective
gathers the RGBA8 bands to the destination rank, which un-permutes them into
the frame.  Every rank holds the frame's visible set (blocks replicated);
`select_visible` is deterministic, so all ranks compute the same list.
"""

from __future__ import annotations

import numpy as np

__all__ = ["part_rows", "assemble", "gather_bands", "render_tiles", "PeerFrame", "render_tiles_fused",
           "BroadcastLoader", "LockstepDone", "shard_blocks", "decode_grid_sharded"]


def part_rows(height: int, band_rows: int, nparts: int, part: int) -> np.ndarray:
    """Frame row indices rendered by `part`, in packed order (afam_frame_rows)."""
    nb = (height + band_rows - 1) // band_rows
    rows = [r for b in range(part, nb, nparts) for r in range(b * band_rows, min(height, (b + 1) * band_rows))]
    return np.asarray(rows, dtype=np.int64)


def assemble(parts, height: int, band_rows: int):
    """Un-permute packed per-part bands into a (height, ...) frame."""
    import torch

    nparts = len(parts)
    first = parts[0]
    frame = torch.empty((height,) + tuple(first.shape[1:]), dtype=first.dtype, device=first.device)
    for p, t in enumerate(parts):
        idx = torch.as_tensor(part_rows(height, band_rows, nparts, p), device=first.device)
        frame.index_copy_(0, idx, t)
    return frame


def gather_bands(local, height: int, band_rows: int, group=None, dst: int = 0):
    """Gather every rank's packed bands to `dst` (NCCL on GPUs, any backend
    on CPU tensors); returns the assembled (height, W, 4) tensor on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return local
    # collectives need equal shapes: pad every part to the largest part's rows
    counts = [len(part_rows(height, band_rows, world, p)) for p in range(world)]
    rmax = max(counts)
    send = local
    if local.shape[0] < rmax:
        send = torch.zeros((rmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    dev = send.device
    if send.is_cuda and dist.get_backend(group) == "gloo":  # gloo gathers host tensors
        send = send.cpu()
    bufs = None
    if rank == dst:
        bufs = [torch.empty_like(send) for _ in range(world)]
    dist.gather(send.contiguous(), bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return assemble([b[:c].to(dev) for b, c in zip(bufs, counts)], height, band_rows)


def render_tiles(pov, blocks: dict, tf, params, *, group=None, band_rows: int = 8, dst: int = 0):
    """render.render across the ranks of `group`: returns the Frame on `dst`
    (None on the other ranks).  Without torch.distributed initialised it is
    a single-GPU render."""
    return submit_tiles(pov, blocks, tf, params, group=group, band_rows=band_rows, dst=dst).result()


def submit_tiles(pov, blocks: dict, tf, params, *, group=None, band_rows: int = 8, dst: int = 0):
    """render_tiles split at the GPU wait (render.PendingFrame): the band
    gather runs in result()."""
    import torch.distributed as dist

    from .render import Frame, PendingFrame, submit_part

    if not (dist.is_available() and dist.is_initialized()):
        return PendingFrame(submit_part(pov, blocks, tf, params, host_out=True), params, render_tiles)
    world, rank = dist.get_world_size(group), dist.get_rank(group)

    def finish(out, info):
        full = gather_bands(out, int(params.height), band_rows, group, dst)
        if full is None:
            return None
        return Frame(int(params.width), int(params.height), full.cpu().numpy())

    return PendingFrame(submit_part(pov, blocks, tf, params, band_rows=band_rows, nparts=world, part=rank),
                        params, render_tiles, finish)


render_tiles.submit = submit_tiles
render_tiles.last_stats = None
render_tiles.frames_in_flight = 2  # per-call output buffers: runtime.replay may keep two frames launched


class PeerFrame:
    """Rank `dst`'s (height, width, 4) uint8 frame buffer mapped into every
    rank of the group over NVLink (CUDA IPC, afam_ipc_*): the fused band
    gather -- each rank's render kernel stores its rows straight into this
    buffer (AFAM_RENDER_FULL_FRAME), so no separate collective moves pixels.
    The handle travels once through torch.distributed."""

    def __init__(self, height: int, width: int, group=None, dst: int = 0, device: int | None = None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib

        self.height, self.width, self.dst = int(height), int(width), int(dst)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nbytes = self.height * self.width * 4
        self._own = self.rank == self.dst
        ptr = C.c_void_p()
        handle, err = None, None
        if self._own:
            try:  # a failure still takes part in the broadcast below, so no rank waits forever
                _lib.check(_lib.lib().afam_device_alloc(self.device, self.nbytes, C.byref(ptr)))
                hb = (C.c_uint8 * 64)()
                _lib.check(_lib.lib().afam_ipc_get_handle(ptr, hb))
                handle = bytes(hb)
            except Exception as exc:  # noqa: BLE001
                err = exc
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            obj = [handle]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, self.dst) if group else self.dst,
                                       group=group, device=torch.device("cuda", self.device)
                                       if dist.get_backend(group) == "nccl" else None)
            handle = obj[0]
            if not self._own:
                if handle is None:
                    raise RuntimeError(f"rank {self.dst} could not export its frame buffer")
                hb = (C.c_uint8 * 64).from_buffer_copy(handle)
                _lib.check(_lib.lib().afam_ipc_open(hb, self.device, C.byref(ptr)))
        if err is not None:
            if ptr.value:
                _lib.lib().afam_device_free(ptr)
            raise err
        self.ptr = int(ptr.value)

    def frame(self):
        """The assembled frame as a host (H, W, 4) uint8 array (rank dst only)."""
        import ctypes as C

        import numpy as np
        import torch

        if not self._own:
            raise RuntimeError("only the destination rank reads the frame")
        from . import _lib

        out = np.empty((self.height, self.width, 4), dtype=np.uint8)
        torch.cuda.synchronize(self.device)
        _lib.check(_lib.lib().afam_copy_to_host(out.ctypes.data_as(C.c_void_p), C.c_void_p(self.ptr), self.nbytes))
        return out

    def close(self):
        from . import _lib

        if self.ptr:
            if self._own:
                _lib.lib().afam_device_free(self.ptr)
            else:
                _lib.lib().afam_ipc_close(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def render_tiles_fused(pov, blocks: dict, tf, params, peer: PeerFrame, *, group=None, band_rows: int = 8):
    """render_tiles with the band gather fused into the render kernel: every
    rank renders its bands (b % world == rank) straight into `peer`, the
    destination rank's frame, over NVLink; one barrier orders the writes
    before the destination reads.  Returns the Frame on the destination rank
    (None elsewhere)."""
    return submit_tiles_fused(pov, blocks, tf, params, peer, group=group, band_rows=band_rows).result()


def submit_tiles_fused(pov, blocks: dict, tf, params, peer: PeerFrame, *, group=None, band_rows: int = 8):
    """render_tiles_fused split at the GPU wait (render.PendingFrame)."""
    import torch.distributed as dist

    from .render import Frame, PendingFrame, submit_part

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0

    def finish(out, info):
        if world > 1:
            dist.barrier(group)  # every rank's kernel (and its peer stores) completed
        if rank != peer.dst:
            return None
        return Frame(int(params.width), int(params.height), peer.frame())

    return PendingFrame(submit_part(pov, blocks, tf, params, band_rows=band_rows, nparts=world, part=rank,
                                    out_ptr=peer.ptr), params, render_tiles_fused, finish)


render_tiles_fused.submit = submit_tiles_fused
render_tiles_fused.last_stats = None
render_tiles_fused.frames_in_flight = 1  # one PeerFrame: a frame is collected before the next is launched


# ------------------------------------------------------------ shared misses
_STATUS = {0: None, 2: "FormatError", 4: "ValueError"}


class LockstepDone:
    """`rendering_done` for a prefetch loop that runs in lockstep on every
    rank: rank 0's answer is broadcast, so every rank stops prefetching
    before the same block (reference runtime.py:183-188 checks
    rendering_done before each load)."""

    def __init__(self, inner, group=None, device=None):
        import torch

        self.inner, self.group = inner, group
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)

    def is_set(self) -> bool:
        import torch.distributed as dist

        if dist.get_rank(self.group) == 0:
            self.flag.fill_(1 if self.inner.is_set() else 0)
        dist.broadcast(self.flag, src=dist.get_global_rank(self.group, 0) if self.group is not None else 0,
                       group=self.group)
        return bool(self.flag.item())


class BroadcastLoader:
    """ModelCache loader for N ranks that share one host store (SURVEY.md
    8e): each cache miss is read from host memory and copied H2D by ONE rank
    (the i-th miss by rank i % N, spreading the PCIe links), then broadcast
    over NVLink (NCCL) into every rank's staging buffer, where
    afam_store_put_mfa_device realigns it into that rank's slot.  The
    reference loads each miss from disk per process (runtime.py:112-133,
    cache_frame :154-166); per-rank H2D (make_loader) stays the default.

    Every rank must issue the same misses in the same order: the cache
    decisions are deterministic given identical histories (select_visible
    is), and replay() wraps the prefetch's rendering_done in LockstepDone
    (`lockstep`) so all ranks stop prefetching at the same block.  Needs a
    render function with `submit` (prefetch on the frame thread)."""

    def __init__(self, manifest, dstore, source, group=None, device=None, max_bytes=None):
        import torch
        import torch.distributed as dist

        from .model import serialized_size

        self.manifest, self.dstore, self.source, self.group = manifest, dstore, source, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.device = torch.device("cuda", dstore.device) if device is None else torch.device(device)
        from . import _lib

        # the largest .mfa image of this store: max_ncp at the largest device degree
        cap = max_bytes if max_bytes is not None else serialized_size(dstore.max_ncp, _lib.AFAM_MAX_DEGREE)
        self.staging = torch.empty(int(cap), dtype=torch.uint8, device=self.device)
        self.hdr = torch.zeros(3, dtype=torch.int64, device=self.device)
        self.misses = 0
        self.h2d_bytes = 0  # bytes this rank copied from the host
        self.recv_bytes = 0  # bytes this rank received over the interconnect

    def _src(self, r):
        import torch.distributed as dist

        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def __call__(self, addr):
        import torch
        import torch.distributed as dist

        from .device import DeviceBlock, check_mfa
        from .errors import FormatError

        ent = self.manifest.entries.get(addr)
        if ent is None:
            raise FormatError(f"manifest has no model file for block {addr.key}")
        root = self.misses % self.world
        self.misses += 1
        buf, msg = None, ""
        if self.rank == root:
            data = self.source(addr)
            buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
            status, deg = 0, 0
            try:
                deg = check_mfa(buf, ent.ncp)
            except FormatError as exc:
                status, msg = 2, str(exc)
            except ValueError as exc:
                status, msg = 4, str(exc)
            self.hdr.copy_(torch.tensor([status, deg, buf.size], dtype=torch.int64))
        dist.broadcast(self.hdr, src=self._src(root), group=self.group)
        status, deg, nbytes = (int(v) for v in self.hdr.tolist())
        if status:
            text = msg or f"block {addr.key}: invalid .mfa image (rank {root})"
            raise FormatError(text) if status == 2 else ValueError(text)
        if nbytes > self.staging.numel():
            raise FormatError(f"block {addr.key}: {nbytes} bytes exceed the staging buffer")
        view = self.staging[:nbytes]
        if self.rank == root:
            view.copy_(torch.from_numpy(np.ascontiguousarray(buf)), non_blocking=True)
            self.h2d_bytes += nbytes
        else:
            self.recv_bytes += nbytes
        dist.broadcast(view, src=self._src(root), group=self.group)
        slot = self.dstore.alloc()
        try:
            st = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
            self.dstore.put_mfa_device(slot, view.data_ptr(), nbytes, deg, ent.ncp, ent.extent, stream=st)
        except Exception:
            self.dstore.release(slot)
            raise
        return DeviceBlock(self.dstore, slot, ent.extent, addr.lod, deg, ent.ncp)

    def release(self, block):
        self.dstore.release(block.slot)

    def sync(self):
        import torch

        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()

    def lockstep(self, done):
        return LockstepDone(done, self.group, self.device)


# ---------------------------------------------------------------------------
# Grid decode over the GPUs of one node (BASELINE config 5):
# MicroModel.decode_grid (model.py:89-93 -> bspline.py:162-172) of every
# block, the blocks dealt round-robin over the ranks.  Blocks are
# independent and the decoded grids stay on their rank, so there is no
# exchange step and no collective.
def shard_blocks(addrs, rank: int | None = None, world: int | None = None, group=None) -> list:
    """This rank's share of a block list: sorted addresses, block i on rank
    i % world (interleaved, so the NCP mix -- and the work -- balances)."""
    if rank is None or world is None:
        import torch.distributed as dist

        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    return sorted(addrs)[rank::world]


def decode_grid_sharded(blocks: dict, m: int, *, group=None, stream=None, rank: int | None = None,
                        world: int | None = None):
    """decode_grid((m, m, m)) of this rank's share of `blocks` ({addr:
    DeviceBlock}, every block resident in one DeviceStore on this rank's GPU)
    in one K3 launch.  Returns (addrs, grids): the rank's addresses and a
    device tensor (n, m, m, m) laid out [b][k][j][i] (x fastest, the decode
    kernels' layout; grids[b].permute(2, 1, 0) is the reference's [i, j, k])."""
    import ctypes as C

    import torch

    from . import _lib
    from .device import stream_handle

    mine = shard_blocks(list(blocks), rank, world, group)
    if not mine:
        return mine, None
    store = blocks[mine[0]].store
    if any(blocks[a].store is not store for a in mine):
        raise ValueError("decode_grid_sharded: the rank's blocks must share one DeviceStore")
    slots = np.ascontiguousarray([blocks[a].slot for a in mine], dtype=np.int32)
    dev = torch.device("cuda", store.device)
    out = torch.empty((len(mine), m, m, m), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().afam_decode_grid(store.handle, slots.ctypes.data_as(C.c_void_p), len(mine), int(m),
                                               C.c_void_p(out.data_ptr()), C.c_void_p(stream_handle(stream, dev))))
    return mine, out
