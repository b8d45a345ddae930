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
    flops = samples * FLOP_VALUE_P3 + shaded * (FLOP_PER_SAMPLE_P3 - FLOP_VALUE_P3)
    achieved = flops / (sum(ktimes) / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "render_kernel_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "fp32", "achieved": achieved, "peak": fma_peak, "unit": "TFLOP/s",
                "frac": achieved / fma_peak if fma_peak else None, "traffic": traffic,
                "kernel": "render_kernel (K2)",
                "note": "algorithmic FLOP (separable p=3 contraction, basis evaluation not credited) = 168 per "
                        "decoded sample (value) + 216 per shaded sample (gradient, TF opacity > 0), over the "
                        "render kernels' device time (CUDA events on the render stream); peak = FFMA "
                        "microbenchmark on this GPU (MEASURED_PEAKS.json has no FP32 figure)",
                "shaded_frac": shaded / max(1, samples)}

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
                             upload_s=round(upload_s, 2), fp64_slot_sample=int(nfp64)),
              "roofline": roofline, "clocks": clk.summary(), "gpu_launches": 3 * args.steps,
              "wall_s_timed_region": t_wall}

    # -- e2e through the public runtime API: ModelCache(200) + linear prefetch, pinned host source
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, man, blobs, povs, tf, params, rank, world, local_rank)
    if peer is not None:
        dist.barrier()
        peer.close()
    del resident_all, ds
    return result, man, blobs


def run_e2e(args, man, blobs, povs, tf, params, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2409_00184_b200 import render, runtime
    from paper_2409_00184_b200.device import DeviceStore

    cap = 200
    ds = DeviceStore(cap + 1, 65, device=local_rank)
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
    draw.samples, draw.d2h = 0, 0
    nwarm = args.warmup
    nsteps = args.e2e_steps or args.steps
    runtime.replay(povs[:nwarm], man, cache, tf, params, prefetch="linear", keep_frames=False, render_fn=draw)
    c0 = cache.counters()
    draw.samples, draw.d2h = 0, 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    timings, _, agg = runtime.replay(povs[nwarm:nwarm + nsteps], man, cache, tf, params, prefetch="linear",
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
    return {"value": float(tot[0]) / float(tot[1]), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": draw.d2h / nsteps, "steps": nsteps,
            "api": "runtime.replay(ModelCache(200), prefetch='linear' on the frame thread while the GPU marches) -> tiles.render_tiles -> Frame bytes on host",
            "mean_caching_ms": agg["mean_caching_ms"], "mean_rendering_ms": agg["mean_rendering_ms"],
            "mean_latency_ms": agg["mean_latency_ms"], "miss_rate": agg["miss_rate"],
            "prefetch_models_loaded": agg["prefetch_models_loaded"]}


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


def host_cpu() -> tuple:
    from oracle import workload

    threads = len(os.sched_getaffinity(0))  # every host core (torchrun sets OMP_NUM_THREADS=1)
    return threads, workload.cpu_model()


def run_reference(args):
    """The reference algorithm on the host CPU: whole 1024^2 frames of the
    config-3 orbit (the same frames as --impl ours: pose W + k), one frame
    per step, the float64 C restatement on every host thread."""
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
