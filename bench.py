"""Benchmark: decoded B-spline samples/s of the 1024^2 ray-cast (BASELINE config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step renders one 1024^2 frame of the config-3 model (1024^3-equivalent
synthetic turbulence: 1025^3 lattice, 4 LODs, 4,680 micro-blocks of 65^3
samples, degree 3, NCP 40..65) from orbit_trajectory(100, radius=2.0)
pose (W + k) % 100, sd = 1e-3, ML transfer function, gradient shading.
`value` = decoded samples / s with every block resident in HBM (device
time, CUDA events on the render stream, L2 flushed between steps, max over
ranks); `e2e` = the same metric through the public runtime API (ModelCache
of 200 blocks + linear prefetch fed from pinned host memory, frame read
back to the host), i.e. BASELINE config 4.  N > 1: one process per GPU
(torchrun), each rank renders interleaved 8-row bands, NCCL gather of
the RGBA8 tiles to rank 0 inside the timed step.

--impl reference times the reference algorithm on the host CPU: the
float64 C restatement in oracle/ (the reference itself is pure Python and
is not on the GPU box), all host threads, one whole frame of the same orbit
per step; it imports nothing from the product package (oracle/workload.py
restates the inputs).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded samples/s (1024^2 ray-cast, config 3)"
DATA = ("synthetic: seeded k^-5/3 turbulence (48 Fourier modes), each block fitted by the reference encoder's "
        "endpoint-pinned least-squares operator at an NCP hash-assigned in [40, 65] (not an adaptive search); "
        "~120 samples per ray under o_max 0.99")
UNIT = "samples/s"
FLOP_PER_SAMPLE_P3 = 384  # 2*(2q^3+3q^2+4q), q=4: separable value+gradient contraction
FLOP_VALUE_P3 = 168  # 2*(q^3+q^2+q): value only (transparent samples skip the gradient, see afam_render.cu)
WORKLOAD = {"workload": "config3: 1024^3-equiv synthetic turbulence, 4 LODs, 4680 blocks (micro 65, degree 3, "
                        "ncp hash-assigned in 40-65), 1024x1024 ray-cast, sd 1e-3, o_max 0.99, ML TF + gradient "
                        "shading, orbit_trajectory(100, r=2.0)",
            "frame": [1024, 1024], "sample_distance": 1e-3, "blocks": 4680,
            "l2": "flushed between steps (512 MiB write outside the per-step events)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="config3", choices=["config3", "config2", "config5"],
                    help="the headline workload; the default config-3 line also carries config 2 and config 5 "
                         "under 'workloads' (unless --no-extra)")
    ap.add_argument("--no-extra", action="store_true", help="config 3 only (no config-2 / config-5 lines)")
    ap.add_argument("--miss-load", default="per-rank", choices=["per-rank", "broadcast"],
                    help="N > 1 e2e: every rank copies its cache misses H2D, or one rank per miss + a broadcast "
                         "over NVLink (tiles.BroadcastLoader)")
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="N > 1: band gather fused into the render kernel (peer stores) or an NCCL gather")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("AFAM_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ data
def build_model(pinned: bool):
    from paper_2409_00184_b200 import synth

    alloc = None
    if pinned:
        import torch

        def alloc(n):
            t = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            alloc.keep = t
            return t.numpy()

    t0 = time.time()
    man, blobs = synth.turbulence_store(alloc=alloc)
    return man, blobs, time.time() - t0


def build_model_distributed(rank, dev):
    """N > 1: rank 0 synthesises the store once; the packed .mfa images are
    broadcast over NVLink (NCCL) and land in every rank's pinned host buffer
    (the e2e path streams blocks from there), so host cores are not shared by
    N copies of the synthesis."""
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import model, synth
    from paper_2409_00184_b200.partition import skeleton

    t0 = time.time()
    man = skeleton(4, 2, 65)
    man.degree = 3
    addrs = sorted(man.entries)
    sizes = [model.serialized_size(synth.ncp_for(a), 3) for a in addrs]
    total = int(sum(sizes))
    host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    if rank == 0:
        man0, _ = synth.turbulence_store(alloc=lambda n: host.numpy())
    dbuf = host.to(dev, non_blocking=False) if rank == 0 else torch.empty(total, dtype=torch.uint8, device=dev)
    dist.broadcast(dbuf, src=0)
    if rank != 0:
        host.copy_(dbuf)
    del dbuf
    arr = host.numpy()
    offs = np.concatenate([[0], np.cumsum(sizes)])
    blobs = {}
    for i, a in enumerate(addrs):
        e = man.entries[a]
        e.ncp, e.nbytes, e.path, e.is_complex = synth.ncp_for(a), sizes[i], a.file_name, True
        blobs[a] = arr[offs[i]:offs[i + 1]]
    build_model_distributed.keep = host
    return man, blobs, time.time() - t0


def measure_fma_peak(dev):
    """FP32 FMA peak of this GPU: a dependent-chain-free FFMA kernel in libafam."""
    import ctypes as C

    import torch

    from paper_2409_00184_b200 import _lib

    out = torch.empty(148 * 8 * 256, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)
    flops = C.c_double()
    best = 0.0
    for _ in range(4):
        ms = C.c_float()
        _lib.check(_lib.lib().afam_bench_fma(C.c_void_p(out.data_ptr()), 4096, C.byref(ms), C.byref(flops),
                                             C.c_void_p(s.cuda_stream)))
        best = max(best, flops.value / (ms.value * 1e-3))
    return best / 1e12


# ------------------------------------------------------------------ ours
def make_peer(args, world, rank, size, local_rank, dev):
    """N > 1: rank 0's frame mapped into every rank (fused band gather), or
    None (NCCL gather) when --gather nccl or when any rank cannot map it."""
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import tiles

    if args.gather != "fused":
        return None
    ok = torch.ones(1, device=dev)
    peer = None
    try:
        peer = tiles.PeerFrame(size, size, device=local_rank)
    except Exception as exc:  # noqa: BLE001
        print(f"rank {rank}: fused gather unavailable ({exc}); using the NCCL gather", file=sys.stderr)
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() < 1:
        if peer is not None:
            peer.close()
        return None
    return peer



def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import render, runtime
    from paper_2409_00184_b200.device import DeviceStore
    from paper_2409_00184_b200.partition import BlockAddress

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world == 1:
        man, blobs, gen_s = build_model(pinned=not args.no_e2e)
    else:
        man, blobs, gen_s = build_model_distributed(rank, dev)
    povs = runtime.orbit_trajectory(100, radius=2.0)
    S = args.size
    params = render.RenderParams(width=S, height=S, sample_distance=1e-3)
    tf = render.TransferFunction.ml_preset()

    # -- every block resident in HBM (the `value` measurement)
    t0 = time.time()
    ds = DeviceStore(len(blobs) + 1, 65, device=local_rank)
    resident_all = {a: ds.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod) for a, b in blobs.items()}
    torch.cuda.synchronize(dev)
    upload_s = time.time() - t0
    nfp64 = sum(ds.info(b.slot)["fp64"] for b in list(resident_all.values())[:: max(1, len(resident_all) // 256)])

    band = 8
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    frame_out = torch.empty((render._lib.lib().afam_frame_rows(S, band, world, rank), S, 4), dtype=torch.uint8,
                            device=dev)
    from paper_2409_00184_b200 import tiles

    # N > 1: the band gather is fused into the render kernel -- every rank
    # stores its pixels straight into rank 0's frame over NVLink (CUDA IPC,
    # tiles.PeerFrame); the NCCL gather is the fallback (or --gather nccl)
    peer = make_peer(args, world, rank, S, local_rank, dev) if world > 1 else None
    gather_kind = "single GPU" if world == 1 else ("fused: peer stores over NVLink" if peer else "NCCL gather")

    def step(k):
        """One frame: render this rank's bands and bring them to rank 0.
        Device time = the render kernels (CUDA events recorded by afam_render
        on the render stream around its launches) + the NCCL gather when the
        gather is not fused (events on the same stream).  Host preparation is
        reported separately."""
        pov = povs[k % len(povs)]
        vis = render.select_visible(pov, man, params.aspect)
        blocks = {a: resident_all[a] for a in vis}
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        if peer is not None:
            _, info, _ = render.render_part(pov, blocks, tf, params, band_rows=band, nparts=world, part=rank,
                                            device=local_rank, out_ptr=peer.ptr)
        else:
            _, info, _ = render.render_part(pov, blocks, tf, params, band_rows=band, nparts=world, part=rank,
                                            device=local_rank, out=frame_out)
        ev1, ev2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev1.record(stream)
        if world > 1 and peer is None:  # NCCL gather of the RGBA8 bands to rank 0 + un-permute there
            tiles.gather_bands(frame_out, S, band)
        ev2.record(stream)
        if peer is not None:
            dist.barrier()  # every rank's kernel (and its peer stores) done before rank 0 uses the frame
        return ev0, ev1, ev2, info, len(vis)

    times, ktimes, envelope, samples, fp64s, shaded, nvis = [], [], [], 0, 0, 0, []
    exact_s, exact_c = 0, 0
    # the sampler starts before the warm-up: nvidia-smi's own start-up must not
    # overlap the timed steps; its samples cover warm-up + timed region (all under load)
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        for k in range(args.warmup):
            step(k)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        if world > 1:
            dist.barrier()
        wall0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()  # evict the previous frame's blocks from L2 (outside the events)
            ev0, ev1, ev2, info, nv = step(args.warmup + k)
            torch.cuda.synchronize(dev)
            ktimes.append(info["kernel_ms"])
            times.append(info["kernel_ms"] + ev1.elapsed_time(ev2))
            envelope.append(ev0.elapsed_time(ev1))
            samples += info["samples"]
            fp64s += info["fp64_samples"]
            shaded += info["shaded_samples"]
            exact_s += info["exact_samples"]
            exact_c += info["exact_cells"]
            nvis.append(nv)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
    # transparent-cell skip: the debug kernel counts the samples that lie in
    # cells whose value range misses the TF's opacity support (counted as
    # decoded -- their TF opacity is provably 0 -- but not contracted); the
    # same frames as the timed steps, outside the timed region
    clear = 0
    for k in range(args.steps):
        pov = povs[(args.warmup + k) % len(povs)]
        vis = render.select_visible(pov, man, params.aspect)
        _, dinfo, _ = render.render_part(pov, {a: resident_all[a] for a in vis}, tf, params, band_rows=band,
                                         nparts=world, part=rank, device=local_rank, debug=True)
        clear += dinfo["clear_samples"]
    step_ms = float(np.mean(times))
    kern_ms = float(np.mean(ktimes))
    tot = torch.tensor([samples, fp64s], dtype=torch.float64, device=dev)
    tmax = torch.tensor([sum(times), sum(ktimes), wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_samples, total_fp64 = float(tot[0]), float(tot[1])
    t_steps, t_kern, t_wall = float(tmax[0]) / 1e3, float(tmax[1]) / 1e3, float(tmax[2])
    value = total_samples / t_steps

    # -- roofline of the dominant kernel (render_kernel)
    fma_peak = measure_fma_peak(dev)
    # the algorithm (reference render.py:445-452) decodes value
    # and gradient for every sample -- 384 FLOP per decoded sample at p = 3.
    # The kernel skips the gradient of samples the TF makes transparent (the
    # frame is bit-identical), so it executes fewer: reported beside it.
    flops = samples * FLOP_PER_SAMPLE_P3
    flops_exec = (samples - clear) * FLOP_VALUE_P3 + shaded * (FLOP_PER_SAMPLE_P3 - FLOP_VALUE_P3)
    achieved = flops / (sum(ktimes) / 1e3) / 1e12
    achieved_exec = flops_exec / (sum(ktimes) / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "render_kernel_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "fp32", "achieved": achieved, "peak": fma_peak, "unit": "TFLOP/s",
                "frac": achieved / fma_peak if fma_peak else None, "traffic": traffic,
                "kernel": "render2_kernel (K2)",
                "note": "algorithmic FLOP per SURVEY.md 8(d): 384 per decoded sample (separable p=3 value + "
                        "gradient contraction, basis evaluation not credited) over the render kernels' device "
                        "time (CUDA events on the render stream); peak = FFMA microbenchmark on this GPU "
                        "(MEASURED_PEAKS.json has no FP32 figure); achieved_executed counts what the kernel "
                        "runs: 168 per sample outside transparent cells + 216 per shaded sample (gradient only "
                        "where TF opacity > 0); samples in transparent cells (clear_sample_frac) run only the "
                        "cell-membership test",
                "achieved_executed": achieved_exec,
                "frac_executed": achieved_exec / fma_peak if fma_peak else None,
                "shaded_frac": shaded / max(1, samples), "clear_sample_frac": clear / max(1, samples)}

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f32 (f64 geometry; f64 decode on "
                                                                 "ill-conditioned blocks)",
              "data": DATA,
              "config": dict(WORKLOAD, parallelism=f"image bands x{world}", gather=gather_kind, frame_ms=step_ms,
                             kernel_ms=kern_ms, host_envelope_ms=float(np.mean(envelope)),
                             visible_blocks_mean=float(np.mean(nvis)),
                             fp64_sample_frac=total_fp64 / max(1.0, total_samples),
                             exact_path_sample_frac=exact_s / max(1, samples),
                             exact_geometry_per_sample=exact_c / max(1, samples), gen_s=round(gen_s, 1),
                             upload_s=round(upload_s, 2), fp64_slot_sample=int(nfp64),
                             empty_space="transparent-cell skip: samples in knot cells whose control-point range "
                                         "(widened by max|c| 2^-14) misses the TF opacity support are counted, not "
                                         "contracted; frames and per-ray sample counts identical to the oracle "
                                         "(tests/test_gpu_cell_skip.py)"),
              "roofline": roofline, "clocks": clk.summary(), "gpu_launches": 3 * args.steps,
              "wall_s_timed_region": t_wall}

    # -- e2e through the public runtime API: ModelCache(200) + linear prefetch, pinned host source
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, man, blobs, povs, tf, params, rank, world, local_rank)
    if peer is not None:
        dist.barrier()
        peer.close()
    del flush
    # -- the other BASELINE configs on the same box (own metric, value and roofline each)
    if not args.no_extra:
        result["workloads"] = {
            "config5": run_config5(ds, resident_all, man, blobs, rank, world, dev, max(3, args.steps // 4),
                                   args.warmup),
            "k1_points": run_k1(ds, resident_all, dev, max(3, args.steps // 4), args.warmup),
            # the same decode on the tcgen05 kernel (3xTF32 x stage), measured beside the default
            "config5_tensor_cores": run_config5(ds, resident_all, man, blobs, rank, world, dev, 3, 1,
                                                path="tensor_cores"),
        }
        del resident_all, ds
        torch.cuda.empty_cache()
        result["workloads"]["config2"] = run_config2(rank, world, dev, args.steps, args.warmup, fma_peak)
    else:
        del resident_all, ds
    return result, man, blobs


def run_headline(args, rank, world, local_rank):
    """--workload config5 / config2: that config's line (value, roofline, e2e)."""
    import torch

    from paper_2409_00184_b200.device import DeviceStore

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    with ClockSampler(local_rank) as clk:
        time.sleep(1.0)
        if args.workload == "config5":
            man, blobs, _ = build_model(pinned=True) if world == 1 else build_model_distributed(rank, dev)
            ds = DeviceStore(len(blobs) + 1, 65, device=local_rank)
            resident_all = {a: ds.load_mfa(b, man.entries[a].ncp, man.entries[a].extent, a.lod)
                            for a, b in blobs.items()}
            torch.cuda.synchronize(dev)
            res = run_config5(ds, resident_all, man, blobs, rank, world, dev, args.steps, args.warmup,
                              e2e=not args.no_e2e)
            res["dtype"] = "f32 (f64 on ill-conditioned blocks)"
        else:
            res = run_config2(rank, world, dev, args.steps, args.warmup, measure_fma_peak(dev),
                              e2e=not args.no_e2e and rank == 0)
            res["dtype"] = "f32 + f64 (ill-conditioned ncp 64/65 blocks decode in float64)"
    res.update({"warmup": args.warmup, "vs_baseline": None, "data": "synthetic (see config.workload)",
                "clocks": clk.summary(), "gpu_launches": None})
    res["gpu_launches"] = args.steps if args.workload == "config5" else 3 * args.steps
    return res


def tiles_mod():
    from paper_2409_00184_b200 import tiles

    return tiles


def run_e2e(args, man, blobs, povs, tf, params, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import render, runtime
    from paper_2409_00184_b200.device import DeviceStore

    cap = 200
    ds = DeviceStore(cap + 1, 65, device=local_rank)
    if world > 1 and args.miss_load == "broadcast":
        loader = tiles_mod().BroadcastLoader(man, ds, lambda a: blobs[a])
    else:
        loader = runtime.make_loader(None, man, ds, source=lambda a: blobs[a])
    cache = runtime.ModelCache(cap, loader)
    band = 8
    S = params.width

    from paper_2409_00184_b200 import tiles

    peer = make_peer(args, world, rank, params.height, local_rank, torch.device("cuda", local_rank)) \
        if world > 1 else None

    def draw(pov, resident, tf_, params_):
        # public API: tiles.render_tiles == render.render on one GPU (N > 1:
        # the fused band gather into rank 0's frame); the Frame (host RGBA8)
        # is the step's result read back to the host
        if peer is not None:
            frame = tiles.render_tiles_fused(pov, resident, tf_, params_, peer, band_rows=band)
            draw.samples += tiles.render_tiles_fused.last_stats["samples"]
        else:
            frame = tiles.render_tiles(pov, resident, tf_, params_, band_rows=band)
            draw.samples += tiles.render_tiles.last_stats["samples"]
        if frame is not None:
            draw.d2h += frame.rgba.nbytes
        return frame

    class Counted:
        # draw split at the GPU wait, so replay prefetches while the GPU marches
        def __init__(self, pending, fn):
            self.pending, self.fn = pending, fn

        def done(self):
            return self.pending.done()

        def result(self):
            frame = self.pending.result()
            draw.samples += self.fn.last_stats["samples"]
            if frame is not None:
                draw.d2h += frame.rgba.nbytes
            return frame

    def submit(pov, resident, tf_, params_):
        if peer is not None:
            return Counted(tiles.submit_tiles_fused(pov, resident, tf_, params_, peer, band_rows=band),
                           tiles.render_tiles_fused)
        return Counted(tiles.submit_tiles(pov, resident, tf_, params_, band_rows=band), tiles.render_tiles)

    draw.submit = submit
    draw.frames_in_flight = 1 if peer is not None else 2  # the fused gather has one frame buffer
    draw.samples, draw.d2h = 0, 0
    # config 4: the whole 100-frame orbit is timed (after W warm-up frames
    # on the same cache, so the first W orbit frames start resident)
    nwarm = args.warmup
    nsteps = args.e2e_steps or len(povs)
    runtime.replay(povs[:nwarm], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
    c0 = cache.counters()
    draw.samples, draw.d2h = 0, 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    timings, _, agg = runtime.replay(povs[:nsteps], man, cache, tf, params, prefetch="linear",
                                     keep_frames=False, render_fn=draw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    el = time.perf_counter() - t0
    c1 = cache.counters()
    tot = torch.tensor([draw.samples, el], dtype=torch.float64, device=torch.device("cuda", local_rank))
    if world > 1:
        s = tot.clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        m = tot.clone()
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        tot = torch.stack([s[0], m[1]])
    h2d = (c1["bytes_loaded"] - c0["bytes_loaded"]) / nsteps
    if peer is not None:
        dist.barrier()
        peer.close()
    extra = {"miss_load": args.miss_load if world > 1 else "single GPU"}
    if hasattr(loader, "h2d_bytes"):
        extra.update(rank_h2d_bytes=loader.h2d_bytes, rank_recv_bytes=loader.recv_bytes)
    if world == 1:
        extra["from_disk"] = e2e_from_disk(man, blobs, povs, tf, params, draw, nwarm, nsteps)
    return {**extra, "value": float(tot[0]) / float(tot[1]), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": draw.d2h / nsteps, "steps": nsteps,
            "api": "runtime.replay over the 100-frame orbit (ModelCache(200), prefetch='linear' on the frame thread "
                   "while the GPU marches, the next frame's caching and launch overlapped with the current frame) -> "
                   "tiles.render_tiles -> Frame bytes on host; wall clock",
            "mean_caching_ms": agg["mean_caching_ms"], "mean_rendering_ms": agg["mean_rendering_ms"],
            "mean_latency_ms": agg["mean_latency_ms"], "miss_rate": agg["miss_rate"],
            "prefetch_models_loaded": agg["prefetch_models_loaded"]}


def e2e_from_disk(man, blobs, povs, tf, params, draw, nwarm, nsteps):
    """The e2e replay with the store on disk, as the reference reads it
    (store.load_model per miss, store.py:33-47): the orbit's blocks are
    written with store.write_store into a temporary directory before the
    timed region (so the page cache is warm), and every miss / prefetch load
    goes through the native file loader (afam_store_put_file: read into
    pinned staging, validate, async H2D)."""
    import shutil
    import tempfile

    import torch

    from paper_2409_00184_b200 import render, runtime, store
    from paper_2409_00184_b200.device import DeviceStore

    need = sorted({a for p in povs for a in render.select_visible(p, man, params.aspect)})
    root = tempfile.mkdtemp(prefix="afam_e2e_store_")
    try:
        t0 = time.perf_counter()
        sub = type(man)(levels=man.levels, micro_dims=man.micro_dims, finest_blocks_per_axis=man.finest_blocks_per_axis,
                        volume_dims=man.volume_dims, bounds=man.bounds, degree=man.degree)
        for a in man.entries:
            sub.entries[a] = man.entries[a]
        store.write_store(root, sub, {a: bytes(blobs[a]) for a in need})
        write_s = time.perf_counter() - t0
        ds = DeviceStore(201, 65)
        cache = runtime.ModelCache(200, runtime.make_loader(root, sub, ds))
        runtime.replay(povs[:nwarm], sub, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
        draw.samples, draw.d2h = 0, 0
        c0 = cache.counters()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, agg = runtime.replay(povs[:nsteps], sub, cache, tf, params, prefetch="linear", keep_frames=False,
                                   render_fn=draw)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        c1 = cache.counters()
        return {"value": draw.samples / el, "unit": UNIT, "steps": nsteps,
                "h2d_bytes_per_step": (c1["bytes_loaded"] - c0["bytes_loaded"]) / nsteps,
                "d2h_bytes_per_step": draw.d2h / nsteps, "mean_caching_ms": agg["mean_caching_ms"],
                "mean_rendering_ms": agg["mean_rendering_ms"], "miss_rate": agg["miss_rate"],
                "store": f"{len(need)} .mfa files (the orbit's blocks) written by store.write_store in "
                         f"{write_s:.2f} s before the timed region (page cache warm); native file loader"}
    finally:
        shutil.rmtree(root, ignore_errors=True)


# ------------------------------------------------------------------ config 5 / config 2
def measured_peaks():
    """(HBM GB/s, source) from MEASURED_PEAKS.json (driver-written), else the
    profiling guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def measure_dfma_peak(dev):
    """FP64 FMA peak of this GPU (afam_bench_dfma)."""
    import ctypes as C

    import torch

    from paper_2409_00184_b200 import _lib

    out = torch.empty(148 * 8 * 256, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    flops = C.c_double()
    best = 0.0
    for _ in range(3):
        ms = C.c_float()
        _lib.check(_lib.lib().afam_bench_dfma(C.c_void_p(out.data_ptr()), 512, C.byref(ms), C.byref(flops),
                                              C.c_void_p(s.cuda_stream)))
        best = max(best, flops.value / (ms.value * 1e-3))
    return best / 1e12


C5_METRIC = "decoded samples/s (decode_grid 65^3 of all 4,680 blocks, config 5)"


def run_config5(ds, resident_all, man, blobs, rank, world, dev, steps, warmup, e2e=False, path="auto"):
    """BASELINE config 5: decode_grid((65,)*3) of every block of the config-3
    model (model.py:89-93 -> bspline.py:162-172), blocks round-robin over the
    ranks (block i on rank i % N: no exchange, the decoded
    grids stay on their rank).  One step = one afam_decode_grid launch over
    this rank's blocks; inputs (2.9 GB of control points) and outputs (5.1 GB
    at N = 1) exceed L2, so no flush is needed.  value = all ranks' samples /
    the max over ranks of the summed device time."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import _lib

    from paper_2409_00184_b200 import tiles

    m = 65
    addrs = tiles.shard_blocks(resident_all, rank, world)  # block i on rank i % N
    slots = np.array([resident_all[a].slot for a in addrs], dtype=np.int32)
    ncps = np.array([resident_all[a].ncp for a in addrs], dtype=np.int64)
    out = torch.empty(len(slots) * m ** 3, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)
    lib = _lib.lib()

    from paper_2409_00184_b200.bspline import DECODE_PATHS

    def launch():
        _lib.check(lib.afam_decode_grid_ex(ds.handle, slots.ctypes.data_as(C.c_void_p), len(slots), m,
                                           C.c_void_p(out.data_ptr()), DECODE_PATHS[path], None,
                                           C.c_void_p(st.cuda_stream)))

    for _ in range(warmup):
        launch()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in evs:
        e0.record(st)
        launch()
        e1.record(st)
    torch.cuda.synchronize(dev)
    ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    t = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_blocks = len(resident_all)
    value = total_blocks * m ** 3 * steps / (float(t[0]) / 1e3)
    nbytes = float((4 * ncps ** 3).sum() + 4 * m ** 3 * len(slots))  # this rank's algorithmic bytes per launch
    hbm, src = measured_peaks()
    achieved = nbytes / (float(np.mean(ms)) * 1e-3) / 1e9
    res = {"metric": C5_METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
           "ms_per_step": float(t[0]) / steps, "higher_is_better": True, "scaling": "strong",
           "config": {"workload": "config5: decode_grid((65,65,65)) of all 4,680 blocks of the config-3 model "
                                  "(ncp hash-assigned in 40-65, degree 3), float32 out",
                      "parallelism": f"blocks round-robin over {world} rank(s), no collective",
                      "blocks_per_rank": len(slots), "l2": "inputs and outputs exceed L2 (2.9 GB in, 5.1 GB out)"},
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                        "frac": achieved / hbm, "traffic": None,
                        "kernel": "decode_tc_kernel (K3, tcgen05 3xTF32 x stage)" if path == "tensor_cores"
                        else "decode_fx_kernel (K3, register-tiled CUDA cores)",
                        "note": "algorithmic bytes = 4 ncp^3 (control points read) + 4 m^3 (grid written) per "
                                f"block, this rank's blocks per launch; peak = {src}"}}
    res["config"]["path"] = path
    if e2e:
        res["e2e"] = config5_e2e(man, blobs, addrs, rank, world, dev, steps)
    del out
    return res


def run_k1(ds, resident_all, dev, steps, warmup):
    """The K1 decode-gather microbenchmark of SURVEY.md 8(d) on the resident
    config-3 store: n = 2^24 parameter points u ~ U[0,1)^3 (default_rng(0)),
    slots uniform over the 4,680 blocks (incoherent gather), value +
    gradient, float32 out (bspline.evaluate_points_with_gradient /
    MicroModel.values_at + gradients_at, model.py:64-87).  HBM roofline with
    the survey's algorithmic bytes per sample (4 q^3 control + 24 point + 4
    slot + 4 value + 12 gradient)."""
    import ctypes as C

    import torch

    from paper_2409_00184_b200 import _lib

    n = 1 << 24
    rng = np.random.default_rng(0)
    slots = np.array([b.slot for b in resident_all.values()], dtype=np.int32)
    u = torch.from_numpy(rng.uniform(0, 1, size=(n, 3))).to(dev)
    sl = torch.from_numpy(slots[rng.integers(0, len(slots), size=n)]).to(dev)
    val = torch.empty(n, dtype=torch.float32, device=dev)
    grad = torch.empty((n, 3), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)
    lib = _lib.lib()

    def launch():
        _lib.check(lib.afam_eval_points(ds.handle, C.c_void_p(sl.data_ptr()), 0, C.c_void_p(u.data_ptr()), n,
                                        C.c_void_p(val.data_ptr()), C.c_void_p(grad.data_ptr()),
                                        _lib.AFAM_EVAL_PARAM, C.c_void_p(st.cuda_stream)))

    for _ in range(warmup):
        launch()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in evs:
        e0.record(st)
        launch()
        e1.record(st)
    torch.cuda.synchronize(dev)
    ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in evs]))
    world = 1
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():  # replicas only: every rank its own batch
        world = dist.get_world_size()
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t[0])
    else:
        ms_max = ms
    per = 4 * 64 + 24 + 4 + 4 + 12
    hbm, src = measured_peaks()
    achieved = n * per / (ms * 1e-3) / 1e9
    return {"metric": "decoded samples/s (K1 point decode, 2^24 incoherent points, value + gradient)",
            "value": world * n / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "config": {"workload": "K1: 2^24 u ~ U[0,1)^3 (default_rng(0)), slots uniform over the 4,680 resident "
                                   "config-3 blocks, AFAM_EVAL_PARAM, value + gradient, float32 out",
                       "parallelism": "replicas: every rank decodes its own 2^24-point batch, no collective",
                       "l2": "the batch's control points (2.9 GB of slots) exceed L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "kernel": "eval_points_grad_kernel (K1)",
                         "note": "algorithmic bytes per sample (SURVEY.md 8d) = 4*4^3 control + 24 point + 4 slot + "
                                 "4 value + 12 gradient; DRAM reads are ~2.2x that (a point's four 64-byte x-quad "
                                 f"runs at 16-byte alignment touch two 64-byte bursts each, profiles/ncu_points_r02.txt); "
                                 f"peak = {src}"}}


def config5_e2e(man, blobs, addrs, rank, world, dev, steps):
    """Config 5 through the C-ABI with host buffers: every step copies this
    rank's .mfa images from pinned host memory (afam_store_put_mfa: H2D +
    realignment on the device), decodes them, and reads the 65^3 grids back
    into pinned host memory; max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import _lib
    from paper_2409_00184_b200.device import DeviceStore
    import ctypes as C

    m = 65
    chunk = 256  # blocks per upload/decode round (device slots reused)
    ds = DeviceStore(chunk, 65, device=dev.index)
    slots = np.array([ds.alloc() for _ in range(chunk)], dtype=np.int32)
    dout = torch.empty(chunk * m ** 3, dtype=torch.float32, device=dev)
    hout = torch.empty(chunk * m ** 3, dtype=torch.float32, pin_memory=True)
    st = torch.cuda.current_stream(dev)
    lib = _lib.lib()

    def one_pass():
        h2d = 0
        for c0 in range(0, len(addrs), chunk):
            part = addrs[c0:c0 + chunk]
            for i, a in enumerate(part):
                ds.put_mfa(int(slots[i]), blobs[a], man.entries[a].ncp, man.entries[a].extent, stream=st)
                h2d += len(blobs[a])
            _lib.check(lib.afam_decode_grid(ds.handle, slots.ctypes.data_as(C.c_void_p), len(part), m,
                                            C.c_void_p(dout.data_ptr()), C.c_void_p(st.cuda_stream)))
            n = len(part) * m ** 3
            hout[:n].copy_(dout[:n], non_blocking=True)
        st.synchronize()
        return h2d

    one_pass()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    nst = max(1, min(steps, 3))
    h2d = 0
    for _ in range(nst):
        h2d += one_pass()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = len(man.entries) * m ** 3 * nst
    return {"value": total / float(t[0]), "unit": UNIT, "h2d_bytes_per_step": h2d / nst,
            "d2h_bytes_per_step": 4 * m ** 3 * len(addrs), "steps": nst,
            "api": "afam_store_put_mfa (pinned .mfa images -> device slots) + afam_decode_grid + D2H of the grids, "
                   f"{chunk}-block rounds, wall clock with a stream sync per step"}


C2_METRIC = "decoded samples/s (512^2 ray-cast, config 2)"
C2_VIEWS = [(0.6, 0.5, 1.2), (2.0, 1.6, 2.6)]


def build_config2():
    from paper_2409_00184_b200 import encoder, synth

    t0 = time.time()
    vol = synth.ml_volume((257, 257, 257))
    man, models, _ = encoder.encode_volume(vol, levels=2, micro_dims=65, degree=3, error_bound=1e-3, coarsest=2,
                                           mode="adaptive")
    return man, models, time.time() - t0


def run_config2(rank, world, dev, steps, warmup, fma_peak, e2e=False):
    """BASELINE config 2: the 257^3 Marschner-Lobb volume encoded adaptively
    (2 LODs, micro 65, degree 3, error bound 1e-3) by the B200 encoder
    (pinned to the reference encoder's decisions, tests/golden/config2.npz),
    512^2 frames at sd 1e-3 alternating between SURVEY.md 8d's two views:
    (0.6, 0.5, 1.2) shows LODs 1 + 2, the three-quarter view (2.0, 1.6, 2.6)
    only LOD-2 blocks, all of them ill-conditioned (ncp 64/65, decoded on the
    float64 path).  N > 1: interleaved 8-row bands per rank, bands stay on
    their rank (no gather)."""
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import render
    from paper_2409_00184_b200.device import DeviceStore

    man, models, enc_s = build_config2()
    params = render.RenderParams(width=512, height=512, sample_distance=1e-3)
    tf = render.TransferFunction.ml_preset()
    ds = DeviceStore(len(models), 65, device=dev.index)
    resident = {a: ds.load_model(mm) for a, mm in models.items()}
    nfp64 = sum(ds.info(b.slot)["fp64"] for b in resident.values())
    povs = [render.PointOfView(np.asarray(p), -np.asarray(p), [0.0, 1.0, 0.0]) for p in C2_VIEWS]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = torch.empty((render._lib.lib().afam_frame_rows(512, 8, world, rank), 512, 4), dtype=torch.uint8,
                      device=dev)

    def frame(k):
        pov = povs[k % 2]
        vis = render.select_visible(pov, man, params.aspect)
        _, info, _ = render.render_part(pov, {a: resident[a] for a in vis}, tf, params, band_rows=8, nparts=world,
                                        part=rank, device=dev.index, out=out)
        return info

    for k in range(warmup):
        frame(k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    kms, samples, s64, shaded, shaded64 = [], 0, 0, 0, 0
    for k in range(steps):
        flush.zero_()
        info = frame(warmup + k)
        kms.append(info["kernel_ms"])
        samples += info["samples"]
        s64 += info["fp64_samples"]
        shaded += info["shaded_samples"]
    tot = torch.tensor([samples, s64, sum(kms)], dtype=torch.float64, device=dev)
    if world > 1:
        t = tot[2:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot[2] = t[0]
    value = float(tot[0]) / (float(tot[2]) / 1e3)
    dfma = measure_dfma_peak(dev)
    # roofline: time the FMA pipes would need for the algorithmic FLOP (value
    # contraction for every sample, + the gradient for shaded ones), float64
    # samples at the FP64 peak and the rest at the FP32 peak, over the
    # measured kernel time (shaded fraction applied uniformly to both kinds)
    f64frac = s64 / max(1, samples)
    flop = samples * FLOP_PER_SAMPLE_P3  # value + gradient per decoded sample
    flop_exec = samples * FLOP_VALUE_P3 + shaded * (FLOP_PER_SAMPLE_P3 - FLOP_VALUE_P3)
    t_ideal = flop * f64frac / (dfma * 1e12) + flop * (1 - f64frac) / (fma_peak * 1e12)
    t_ideal_exec = flop_exec * f64frac / (dfma * 1e12) + flop_exec * (1 - f64frac) / (fma_peak * 1e12)
    t_meas = sum(kms) / 1e3
    res = {"metric": C2_METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
           "ms_per_step": float(tot[2]) / steps, "higher_is_better": True, "scaling": "strong",
           "config": {"workload": "config2: 257^3 Marschner-Lobb, encoded adaptively by the B200 encoder "
                                  "(levels 2, micro 65, degree 3, error bound 1e-3; reference decisions), 512x512 "
                                  "ray-cast, sd 1e-3, o_max 0.99, ML TF + shading, views (0.6,0.5,1.2) / "
                                  "(2.0,1.6,2.6) alternating",
                      "blocks": len(models), "fp64_slots": int(nfp64), "encode_s": round(enc_s, 1),
                      "fp64_sample_frac": float(tot[1]) / max(1.0, float(tot[0])),
                      "parallelism": f"image bands x{world} (bands stay on their rank)",
                      "l2": "flushed between steps (512 MiB write outside the per-step events)"},
           "roofline": {"bound": "fp64+fp32", "achieved": flop / t_meas / 1e12, "peak": dfma, "unit": "TFLOP/s",
                        "frac": t_ideal / t_meas, "traffic": None, "kernel": "render kernels (K2, float64 path)",
                        "note": f"frac = (float64 samples' algorithmic FLOP at the measured FP64 FMA peak {dfma:.1f} "
                                f"TFLOP/s + float32 samples' at the FP32 peak {fma_peak:.1f}) / kernel time; "
                                "384 FLOP per decoded sample (SURVEY.md 8(d), as config 3); frac_executed: the "
                                "kernel's own count (168 value + 216 gradient when shaded)",
                        "frac_executed": t_ideal_exec / t_meas}}
    if e2e:
        res["e2e"] = config2_e2e(man, models, povs, tf, params, rank, world, dev, steps)
    return res


def config2_e2e(man, models, povs, tf, params, rank, world, dev, steps):
    """Config 2 through the public API with host models (the reference CLI's
    call, cli.py:153-164): render.render(pov, {addr: MicroModel}, tf, params)
    uploads the visible blocks (H2D + realignment on the device) and returns
    the host Frame.  Every step gets fresh model objects (shallow copies made
    before the timed region), so every step uploads its whole visible set.
    Rank 0 only at N > 1 (render.render draws whole frames)."""
    import copy

    import torch

    from paper_2409_00184_b200 import model as mmod
    from paper_2409_00184_b200 import render

    sets = []
    for k in range(steps + 1):
        pov = povs[k % 2]
        vis = render.select_visible(pov, man, params.aspect)
        sets.append((pov, {a: copy.copy(models[a]) for a in vis}))

    def one(k):
        pov, blocks = sets[k]
        fr = render.render(pov, blocks, tf, params)
        h2d = sum(mmod.serialized_size(b.ncp, b.degree) for b in blocks.values())
        return render.render.last_stats["samples"], fr.rgba.nbytes, h2d

    one(0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    tot, d2h, h2d = 0, 0, 0
    for k in range(1, steps + 1):
        s, o, i = one(k)
        tot += s
        d2h += o
        h2d += i
    el = time.perf_counter() - t0
    return {"value": tot / el, "unit": UNIT, "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": d2h / steps,
            "steps": steps, "api": "render.render(pov, {addr: MicroModel}, tf, params) -> Frame (host RGBA8); "
                                   "fresh host models every step, so every visible block is uploaded per frame"}


# ------------------------------------------------------------------ CPU
def cpu_frame(frame_index: int, size: int, threads: int, rows=None):
    """Render one orbit frame of the config-3 model with the float64 C
    restatement of render.py:398-466 (oracle/), on `threads` host threads.
    Product-free: the visible set comes from oracle.select_visible and the
    visible blocks' .mfa images from oracle/workload.py (byte-identical to
    the product's synthesis), so the reference arm maps no libafam code.
    Returns (samples, seconds of the render call, description)."""
    from oracle import oracle, workload

    povs = workload.orbit_trajectory(100, radius=2.0)
    pov = povs[frame_index % len(povs)]
    params = workload.render_params(width=size, height=size, sample_distance=1e-3)
    tf = workload.ml_preset()
    man = workload.skeleton(4, 2, 65)
    vis = [workload.Addr(v[0], tuple(v[1:])) for v in oracle.select_visible(pov, man, params.aspect)]
    man, blobs = workload.turbulence_store(addrs=vis)
    host = {a: workload.parse_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod) for a in vis}
    t0 = time.perf_counter()
    _, info = oracle.render(pov, host, tf, params, rows=rows, nthreads=threads)
    el = time.perf_counter() - t0
    what = f"orbit frame {frame_index % len(povs)}" + ("" if rows is None else f" rows {rows[0]}..{rows[1]}")
    return info["samples"], el, what


def cpu_baseline_other(workload: str) -> dict:
    """The oracle on the host cores for --workload config5 (decode_grid of a
    sample of blocks, one block per thread) / config2 (a 64-row band of the
    first view)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle, workload as wl

    threads, model = host_cpu()
    if workload == "config5":
        man = wl.skeleton(4, 2, 65)
        addrs = sorted(man.entries)[:: 4680 // (2 * threads)][: 2 * threads]
        man, blobs = wl.turbulence_store(addrs=addrs)
        ctrls = [wl.parse_mfa(blobs[a], man.entries[a].ncp, man.entries[a].extent, a.lod).control for a in addrs]
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda c: oracle.decode_grid(c, 3, 65), ctrls))
        el = time.perf_counter() - t0
        return {"value": len(ctrls) * 65 ** 3 / el, "unit": UNIT, "cores": threads, "kind": "port", "cpu": model,
                "sample": f"decode_grid((65,)*3) of {len(ctrls)} config-5 blocks in {el:.1f} s (oracle/ C float64, "
                          f"one block per thread, {threads} threads, {model})"}
    from paper_2409_00184_b200 import render

    man, models, _ = build_config2()
    p = np.asarray(C2_VIEWS[0])
    pov = render.PointOfView(p, -p, [0.0, 1.0, 0.0])
    params = render.RenderParams(width=512, height=512, sample_distance=1e-3)
    vis = render.select_visible(pov, man, params.aspect)
    t0 = time.perf_counter()
    _, info = oracle.render(pov, {a: models[a] for a in vis}, render.TransferFunction.ml_preset(), params,
                            rows=(224, 288), nthreads=threads)
    el = time.perf_counter() - t0
    return {"value": info["samples"] / el, "unit": UNIT, "cores": threads, "kind": "port", "cpu": model,
            "sample": f"rows 224..288 of the (0.6,0.5,1.2) 512^2 frame: {info['samples']} samples in {el:.1f} s "
                      f"(oracle/ C float64, OpenMP x{threads}, {model})"}


def host_cpu() -> tuple:
    from oracle import workload

    threads = len(os.sched_getaffinity(0))  # every host core (torchrun sets OMP_NUM_THREADS=1)
    return threads, workload.cpu_model()


def run_reference(args):
    """The reference algorithm on the host CPU: whole 1024^2 frames of the
    config-3 orbit (the same frames as --impl ours: pose W + k), one frame
    per step, the float64 C restatement on every host thread."""
    if args.workload == "config5":
        cb = cpu_baseline_other("config5")
        return {"metric": C5_METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": 0, "steps": 1,
                "warmup": 0, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-3 model)",
                "config": {"workload": "config5: decode_grid((65,65,65)) of a sample of the 4,680 config-3 blocks"},
                "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.workload == "config2":
        return {"impl": "reference", "unavailable": "config 2's encoded store comes from the B200 encoder; "
                                                    "the reference arm is timed on config 3 / config 5"}
    threads, model = host_cpu()
    for k in range(min(args.warmup, 1)):
        cpu_frame(k, args.size, threads)
    tot_s, tot_t = 0, 0.0
    frames = []
    for k in range(args.steps):
        s, t, what = cpu_frame(args.warmup + k, args.size, threads)
        tot_s += s
        tot_t += t
        frames.append(what)
    value = tot_s / tot_t
    sample = (f"whole {args.size}x{args.size} frames, one per step ({frames[0]} .. {frames[-1]}); oracle/ C float64 "
              f"restatement of render.py:398-466, OpenMP x{threads} on {threads} host threads ({model})")
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": DATA, "config": dict(WORKLOAD, l2="n/a (CPU)"),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu": model,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    import torch
    import torch.distributed as dist

    if os.environ.get("AFAM_BENCH_SAME_GPU"):  # functional N>1 check on a 1-GPU box (gloo)
        local_rank = 0
    if world > 1:
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("AFAM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    if args.workload != "config3":
        res = run_headline(args, rank, world, local_rank)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline_other(args.workload)
        if rank == 0:
            print(json.dumps(res), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    res, man, blobs = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads, model = host_cpu()
        s, t, what = cpu_frame(args.warmup, args.size, threads)
        res["cpu_baseline"] = {"value": s / t, "unit": UNIT, "cores": threads, "kind": "port", "cpu": model,
                               "sample": f"one whole {args.size}x{args.size} frame ({what}): {s} samples in {t:.1f} s "
                                         f"(oracle/ C float64, OpenMP x{threads}, {model})"}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
