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

__all__ = ["part_rows", "assemble", "gather_bands", "render_tiles"]


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
    import torch.distributed as dist

    from .render import Frame, render_part

    if not (dist.is_available() and dist.is_initialized()):
        out, info, _ = render_part(pov, blocks, tf, params, host_out=True)
        render_tiles.last_stats = info
        return Frame(int(params.width), int(params.height), out.numpy())
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    out, info, _ = render_part(pov, blocks, tf, params, band_rows=band_rows, nparts=world, part=rank)
    render_tiles.last_stats = info
    full = gather_bands(out, int(params.height), band_rows, group, dst)
    if full is None:
        return None
    return Frame(int(params.width), int(params.height), full.cpu().numpy())


render_tiles.last_stats = None
