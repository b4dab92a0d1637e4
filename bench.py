"""Benchmark: multi-ring allreduce bus GB/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...            (N > 1)

Workload (config 2 of BASELINE.json): a 25,600,000-element fp32 buffer per
rank (ResNet-50 gradient size, 102.4 MB), synthetic inputs from the reference's
own generator (`generate_input`, seed 0).
* N = 1: the 8 ranks of config 2 (grid 2x2x2) live on the one GPU and the
  local-reduce kernel (mode "local") folds every owned region from the 8
  buffers in the reference order and writes all 8 -- the HBM roofline of the
  path.  busbw is reported per (virtual) rank.
* N > 1: one process per GPU, grid (2,), (2,2) or (2,2,2) for N = 2/4/8, the
  multi-GPU kernel over NVLink-mapped peer memory (mode --mode, default auto).

Metric definitions (NCCL convention): algbw = S/t,
busbw = 2(R-1)/R * S / t for R ranks.  `value` = busbw summed over the
physical GPUs (N * busbw; at N = 1 the single GPU's busbw).  Every step
restores the inputs and flushes L2 (256 MiB write, read back so no dirty
lines are charged to the kernel) outside the timed region; the timed region
is one allreduce, CUDA events on the launching stream, max over ranks.
At N > 1 the line also carries `curve`: busbw at 4 KB, 64 KB, 1 MB, 16 MB,
256 MB and 1 GiB per rank (the metric's "vs msg size"), timed the same way, and
`reduce_scatter` / `allgather` on the config buffer (busbw = (N-1)/N * S / t).
`--impl reference` runs the reference runtime's phase loop ported to C
(oracle/rbx_oracle.c, one thread per rank) on the host on the same job.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ELEM = 25_600_000
NOMINAL_NVLINK_GBS = 900.0
MEASURED_PEER_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (NVLink reference)
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
DIMS_FOR = {1: (2, 2, 2), 2: (2,), 4: (2, 2), 8: (2, 2, 2)}
CURVE_BYTES = (4096, 65536, 1 << 20, 16 << 20, 256 << 20, 1 << 30)  # N>1 busbw-vs-size points in the bench line
SPIN_CYCLES = int(os.environ.get("BENCH_SPIN_CYCLES", "1000000"))


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--mode", default="auto", help="auto|fused|fused_pull|ring_dims (N>1)")
    p.add_argument("--dims", default=None, help="grid, e.g. 2x4 (default: 2x2x2 / 2x2 / 2)")
    p.add_argument("--elems", type=int, default=N_ELEM)
    p.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-nccl", action="store_true")
    p.add_argument("--curve", type=int, default=1, help="N>1: add busbw at 4 KB..1 GiB to the line")
    p.add_argument("--e2e-chunks", type=int, default=None,
                   help="N=1: pipeline windows of the host-buffer e2e leg (default 12, best measured against the "
                        "host PCIe ceiling, profiles/r02_e2e_probe_align_1gpu.jsonl); N>1 uses the runtime's default")
    a = p.parse_args()
    if a.e2e_chunks is None:
        a.e2e_chunks = 12 if a.gpus == 1 else None  # N>1: hoststage.default_windows
    return a


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def bind_host_to_gpu(index: int) -> list:
    """Pin this process to the CPU cores NVML reports as local to GPU `index`
    (its PCIe root's NUMA node), so pinned host buffers for the e2e leg are
    allocated and copied near the GPU.  Returns the cores, or [] if unknown."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cores = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
        cores = [c for c in cores if c < os.cpu_count()]
        if cores:
            os.sched_setaffinity(0, cores)
        return cores
    except Exception:  # noqa: BLE001 -- best effort (no NVML / no permission)
        return []


def flush_l2(scratch):
    """Evict L2: write a 256 MiB buffer (> 126 MB L2), then read it back so the
    dirty lines are written back before the timed region starts (otherwise
    their write-back would be charged to the kernel being timed)."""
    import torch

    scratch.fill_(1.0)
    scratch.sum()
    # device spin (default 1M cycles, ~0.5 ms; env BENCH_SPIN_CYCLES) so the host
    # enqueues the timed launch before the GPU gets there: the events then time
    # the kernel, not Python launch latency
    torch.cuda._sleep(SPIN_CYCLES)


def host_link_ms(pairs, dev, stream, iters=5, before=None):
    """The host link's ceiling for the e2e step, measured in the same run: the same bytes
    copied H2D and D2H at the same time on two streams (pinned memory, no kernel).
    pairs: [(pinned host tensor, device tensor)]; returns the median ms."""
    import torch

    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    back = [torch.empty_like(h).pin_memory() for h, _ in pairs]
    scratch_dev = [torch.empty_like(d) for _, d in pairs]
    ts = []
    for _ in range(iters):
        if before:
            before()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        s_in.wait_event(s)
        s_out.wait_event(s)
        with torch.cuda.stream(s_in):
            for (h, _), d in zip(pairs, scratch_dev):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s_out):
            for (_, d), b in zip(pairs, back):
                b.copy_(d, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def workload_name(n: int, dtype: str, ranks: int, dims) -> str:
    """Same string on every arm (ours / --impl reference) for the same job."""
    return f"config2: {n} {dtype}/rank, {ranks} ranks, grid {'x'.join(map(str, dims))}"


def busbw(ranks: int, nbytes: int, seconds: float) -> float:
    return 2.0 * (ranks - 1) / ranks * nbytes / seconds / 1e9


def cpu_port_run(dims, n, steps=None, budget_s=12.0, seed=0):
    """The reference runtime's phase loop ported to C (oracle/, one thread per
    rank) on this host's cores -- the CPU baseline ("kind": "port")."""
    import numpy as np

    from oracle import oracle_c
    from oracle import ringbox_oracle as orc

    ranks = 1
    for d in dims:
        ranks *= d
    parts = [orc.generate_input(seed, 0, r, n, "f32") for r in range(ranks)]
    times = []
    t_end = time.time() + budget_s
    while True:
        bufs = [p.copy() for p in parts]
        times.append(oracle_c.runtime_port(dims, bufs, "f32"))
        if steps is not None and len(times) >= steps:
            break
        if steps is None and (time.time() > t_end and len(times) >= 2):
            break
    del np
    return times, ranks


def run_reference(args):
    """--impl reference: the reference's CPU multi-ring allreduce (C port of
    its runtime phase loop, one thread per rank) on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_gpus = args.gpus
    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else DIMS_FOR.get(n_gpus, (n_gpus,))
    times, ranks = cpu_port_run(dims, args.elems, steps=args.warmup + args.steps)
    timed = times[args.warmup:]
    t = statistics.mean(timed)
    nbytes = args.elems * 4
    bw = busbw(ranks, nbytes, t)
    value = bw  # per-(virtual-)GPU bus bandwidth, the same definition as the GPU arm's `value`
    cores = len(os.sched_getaffinity(0))
    line = {
        "metric": "multi-ring allreduce bus GB/s vs msg size at 2/4/8 B200; % of 900 GB/s NVLink",
        "impl": "reference", "value": round(value, 4), "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generate_input, seed 0)",
        "config": {"workload": workload_name(args.elems, "f32", ranks, dims), "placement": f"CPU, {ranks} threads",
                   "ranks": ranks, "dims": list(dims), "bytes_per_rank": nbytes,
                   "value_definition": "per-rank busbw = 2(R-1)/R*S/t (NCCL convention), t = one full allreduce"},
        "aggregate_busbw_gbs": round(bw * ranks, 4),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": min(ranks, cores), "kind": "port",
                         "sample": f"{args.steps} full allreduces of {args.elems} fp32 x {ranks} ranks "
                                   f"(oracle/rbx_oracle.c orc_runtime_port, {ranks} threads, host has {cores} cores)"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main_single(args):
    """N = 1: the 8 ranks of config 2 on one GPU, local-reduce kernel."""
    import numpy as np
    import torch

    from paper_1708_02188_b200.runtime import Workload, generate_input
    from paper_1708_02188_b200.virtual import VirtualRanks

    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else DIMS_FOR[1]
    ranks = 1
    for d in dims:
        ranks *= d
    n = args.elems
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    bind_host_to_gpu(0)
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esz = 4 if args.dtype == "f32" else 2
    wl = Workload(lengths=(n,), dtype="f32", seed=0)  # the reference's inputs (runtime.py:94-100)
    host = [torch.from_numpy(generate_input(wl, 0, r, n)).to(tdt) for r in range(ranks)]
    pristine = [h.to(dev) for h in host]
    work = [torch.empty_like(p) for p in pristine]
    scratch = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)
    vr = VirtualRanks(dims, device=0)
    stream = torch.cuda.current_stream(dev)

    def restore():
        for w, p in zip(work, pristine):
            w.copy_(p)
        flush_l2(scratch)  # flush L2

    # correctness of the exact timed configuration (one check, outside timing)
    restore()
    vr.collective(work, mode="local")
    torch.cuda.synchronize()
    vr.check()

    for _ in range(args.warmup):
        restore()
        vr.collective(work, mode="local")
    torch.cuda.synchronize()

    sampler = ClockSampler(0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = vr.launches
    sampler.start()
    torch.cuda.synchronize()
    for s, e in ev:
        restore()
        s.record(stream)
        vr.collective(work, mode="local")
        e.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = vr.launches - l0
    vr.check()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    t = statistics.mean(step_ms) / 1e3
    nbytes = n * esz
    bw = busbw(ranks, nbytes, t)

    # e2e through the product API with HOST buffers (VirtualRanks.allreduce_host: the
    # numpy arrays page-locked once, H2D / kernel / D2H of element windows overlapped
    # on three streams) -- every byte crosses PCIe both ways inside the timed region
    e2e_ms, e2e_ok = [], False
    if args.dtype == "f32":
        from paper_1708_02188_b200.runtime import host_empty

        arrays = [host_empty(n, "f32") for _ in host]  # page-locked host buffers (runtime.host_empty)
        for it in range(args.warmup + max(3, min(args.steps, 10))):
            for a, h in zip(arrays, host):
                a[...] = h.numpy()
            flush_l2(scratch)
            s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_ev.record(stream)
            vr.allreduce_host(arrays, mode="local", windows=args.e2e_chunks)
            e_ev.record(stream)
            torch.cuda.synchronize()
            if it >= args.warmup:
                e2e_ms.append(s_ev.elapsed_time(e_ev))
        restore()
        vr.collective(work, mode="local")
        torch.cuda.synchronize()
        e2e_ok = all(np.array_equal(a, w.cpu().numpy()) for a, w in zip(arrays[:2], work[:2]))
    t_e2e = statistics.mean(e2e_ms) / 1e3 if e2e_ms else None
    hl = host_link_ms([(h.pin_memory(), w) for h, w in zip(host, work)], dev, stream,
                      before=lambda: flush_l2(scratch)) if e2e_ms else None

    peak, peak_src = hbm_peak()
    hbm_bytes = 2 * ranks * nbytes  # read every rank buffer once, write every rank buffer once
    achieved = hbm_bytes / t / 1e9
    workload = workload_name(n, args.dtype, ranks, dims)
    traffic = ncu_traffic("local_2x2x2_25.6M_f32") if (dims == (2, 2, 2) and n == N_ELEM and args.dtype == "f32") else None

    cpu = None
    if not args.no_cpu_baseline:
        times, r_ = cpu_port_run(dims, n, budget_s=10.0)
        tc = statistics.median(times)
        cores = len(os.sched_getaffinity(0))
        cpu = {"value": round(busbw(ranks, n * 4, tc), 4), "unit": "GB/s", "cores": min(ranks, cores), "kind": "port",
               "sample": f"{len(times)} full allreduces of config 2 ({n} fp32 x {ranks} ranks, grid "
                         f"{'x'.join(map(str, dims))}) with the C port of the reference runtime, one thread per rank; "
                         f"median {tc * 1e3:.1f} ms; host has {cores} cores"}

    line = {
        "metric": "multi-ring allreduce bus GB/s vs msg size at 2/4/8 B200; % of 900 GB/s NVLink",
        "value": round(bw, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (reference generate_input, seed 0)",
        "config": {"workload": workload, "placement": "1 GPU: all ranks' buffers in HBM, local-reduce kernel",
                   "ranks": ranks, "dims": list(dims), "bytes_per_rank": nbytes,
                   "mode": "local", "l2": "flushed between steps (256 MiB write) and inputs 819 MB > L2",
                   "value_definition": "busbw = 2(R-1)/R*S/t per (virtual) rank; 1 GPU"},
        "busbw_gbs": round(bw, 3), "algbw_gbs": round(nbytes / t / 1e9, 3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": hbm_bytes},
        "cpu_baseline": cpu,
        "e2e": None if t_e2e is None else {
            "value": round(busbw(ranks, nbytes, t_e2e), 4), "unit": "GB/s",
            "h2d_bytes_per_step": ranks * nbytes, "d2h_bytes_per_step": ranks * nbytes,
            "ms_per_step": round(t_e2e * 1e3, 3), "windows": args.e2e_chunks, "result_matches_device_path": e2e_ok,
            "host_link_ms": round(hl, 3), "frac_of_host_link": round(hl / (t_e2e * 1e3), 4),
            "api": "VirtualRanks.allreduce_host on runtime.host_empty numpy buffers (page-locked), 3-stream window pipeline"},
        "gpu_launches": launches,
        "clocks": clocks,
        "step_ms": [round(x, 4) for x in step_ms],
    }
    print(json.dumps(line), flush=True)


def main_multi(args):
    """N > 1: one process per GPU (torchrun, or self-launched by main()).  The
    line's `value` is the per-GPU bus bandwidth of the config buffer (the
    metric: bus GB/s per GPU and % of 900); the job aggregate is reported as
    `aggregate_busbw_gbs`."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import PlacedBuffer, RankContext, Workload, allreduce, generate_input

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # one rank per GPU; a box with fewer GPUs than ranks (a functional check of the
    # N-rank path only, timings meaningless) shares GPUs and uses gloo for the host side
    ngpu = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", rank)) % ngpu
    shared = world > ngpu
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    bind_host_to_gpu(local)
    if shared:
        dist.init_process_group("gloo")
        args.no_nccl = True
    else:
        dist.init_process_group("nccl", device_id=dev)
    dims = tuple(int(x) for x in args.dims.split("x")) if args.dims else DIMS_FOR.get(world, (world,))
    grid = Grid(dims)
    assert grid.size == world, f"dims {dims} do not match world size {world}"
    n = args.elems
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esz = 4 if args.dtype == "f32" else 2
    nbytes = n * esz
    ctx = RankContext(rank, grid, device=local, mode=args.mode, blocking=False)
    host_np = generate_input(Workload(lengths=(n,), dtype="f32", seed=0), 0, rank, n)
    host = torch.from_numpy(host_np).to(tdt)
    pristine = host.to(dev)
    work = ctx.empty(n, args.dtype)
    scratch = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def restore():
        work.copy_(pristine)
        flush_l2(scratch)

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def timed(c, fn, iters, before):
        """before() (restore / L2 flush, ends with a device spin so the host runs
        ahead), a device flag barrier, then fn() between CUDA events on the
        launching stream; per-iteration max over ranks, in ms."""
        ev = []
        for _ in range(iters):
            before()
            c.barrier()  # device-side: the ranks leave it together
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            ev.append((s, e))
        torch.cuda.synchronize()
        c.check()
        return max_over_ranks([s.elapsed_time(e) for s, e in ev])

    # correctness of the exact timed configuration (outside timing)
    restore()
    ctx.collective("allreduce", work)
    ctx.synchronize()
    timed(ctx, lambda: ctx.collective("allreduce", work), args.warmup, restore)
    dist.barrier()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    l0 = ctx.launches
    step_ms = timed(ctx, lambda: ctx.collective("allreduce", work), args.steps, restore)
    launches = ctx.launches - l0 - args.steps  # minus the barrier launches (outside the timed region)
    clocks = sampler.stop() if rank == 0 else None
    t = statistics.mean(step_ms) / 1e3
    bw = busbw(world, nbytes, t)

    # the same collective replayed from a CUDA graph (how a training step captured whole runs it,
    # dp.MultiringDataParallel.capture): capture once, time replays the same way
    graph_replay = None
    try:
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            ctx.collective("allreduce", work)
        stream.wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ctx.collective("allreduce", work)
        gms = timed(ctx, graph.replay, 3, restore)
        gms = timed(ctx, graph.replay, max(5, min(args.steps, 10)), restore)
        gt = statistics.mean(gms) / 1e3
        graph_replay = {"us": round(gt * 1e6, 2), "busbw_gbs": round(busbw(world, nbytes, gt), 2)}
        del graph
    except Exception as exc:  # noqa: BLE001 -- reported, not fatal
        graph_replay = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # the other grids of the same box size on the same buffer: config 1 (2x4) at N=8, (4,) at N=4
    other = {}
    for odims in {8: [(2, 4), (8,)], 4: [(4,)]}.get(world, []):
        if odims == dims:
            continue
        octx = RankContext(rank, Grid(odims), device=local, mode=args.mode, blocking=False)
        owork = octx.empty(n, args.dtype)

        def orestore(w=owork):
            w.copy_(pristine)
            flush_l2(scratch)

        timed(octx, lambda c=octx, w=owork: c.collective("allreduce", w), 3, orestore)
        ms = timed(octx, lambda c=octx, w=owork: c.collective("allreduce", w), max(5, min(args.steps, 10)), orestore)
        ot = statistics.mean(ms) / 1e3
        other["x".join(map(str, odims))] = {"us": round(ot * 1e6, 2), "busbw_gbs": round(busbw(world, nbytes, ot), 2)}
        octx.close()

    # NVLink ceiling on this box, measured in the same run: every rank pushes the allreduce's
    # bus bytes (2(N-1)/N * S per GPU, 2S/N to each peer) into every peer's copy of a registered
    # buffer with the copy engines (cudaMemcpyAsync, one stream per peer), all ranks at once --
    # the fastest engine in profiles/r02_nvlink_ceiling_*.jsonl, no fold, no ordering
    ceiling = None
    if not shared:
        try:
            from cuda.bindings import runtime as cr

            per_peer = (2 * nbytes // world) // 256 * 256
            cbuf = ctx.empty(per_peer * world // 4 + 64, "f32")
            peers = [q for q in range(world) if q != rank]
            streams = [torch.cuda.Stream(dev) for _ in peers]
            my = cbuf.data_ptr()

            def push():
                start = torch.cuda.Event()
                start.record(stream)
                for q, st in zip(peers, streams):
                    st.wait_event(start)
                    dst = ctx.peer_pointer(cbuf, q) + rank * per_peer
                    cr.cudaMemcpyAsync(dst, my + q * per_peer, per_peer, cr.cudaMemcpyKind.cudaMemcpyDefault,
                                       st.cuda_stream)
                for st in streams:
                    stream.wait_stream(st)

            timed(ctx, push, 3, lambda: flush_l2(scratch))
            cms = timed(ctx, push, 10, lambda: flush_l2(scratch))
            ct = statistics.median(cms) / 1e3
            ceiling = {"gbs_per_direction": round(2 * (world - 1) / world * nbytes / ct / 1e9, 1),
                       "us": round(ct * 1e6, 2), "bytes_per_direction": int(per_peer * (world - 1)),
                       "engine": "copy engines: cudaMemcpyAsync push of 2S/N to every peer, one stream per peer, "
                                 "all ranks at once (no fold, no ordering)"}
            del cbuf
        except Exception as exc:  # noqa: BLE001 -- cuda-python missing: report the recipe's figure
            ceiling = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # e2e through the product API with a HOST buffer: runtime.allreduce(ctx, PlacedBuffer(numpy))
    # -- page-locked once, H2D / kernel / D2H of element windows on three streams; every step
    # copies the whole buffer in and the result out inside the timed region (device events)
    e2e = None
    if args.dtype == "f32":
        from paper_1708_02188_b200.runtime import host_empty

        arr = host_empty(n, "f32")  # page-locked host buffer (runtime.host_empty)
        ems = []
        for it in range(args.warmup + max(3, min(args.steps, 10))):
            arr[...] = host_np
            flush_l2(scratch)
            ctx.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            allreduce(ctx, PlacedBuffer(arr, memory="host"))
            e.record(stream)
            torch.cuda.synchronize()
            if it >= args.warmup:
                ems.append(s.elapsed_time(e))
        ems = max_over_ranks(ems)
        t_e2e = statistics.mean(ems) / 1e3
        restore()
        ctx.collective("allreduce", work)
        ctx.synchronize()
        ok = torch.tensor([1 if np.array_equal(arr, work.cpu().numpy()) else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        hl = max_over_ranks([host_link_ms([(host.pin_memory(), work)], dev, stream,
                                          before=lambda: (flush_l2(scratch), ctx.barrier()))])[0]
        e2e = {"value": round(busbw(world, nbytes, t_e2e), 3), "unit": "GB/s",
               "host_link_ms": round(hl, 3), "frac_of_host_link": round(hl / (t_e2e * 1e3), 4),
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": round(t_e2e * 1e3, 3),
               "aggregate_gbs": round(busbw(world, nbytes, t_e2e) * world, 3),
               "result_matches_device_path": bool(ok.item()),
               "api": "runtime.allreduce(ctx, PlacedBuffer(numpy from runtime.host_empty)): page-locked host buffer, 3-stream window pipeline"}

    # the metric's "vs msg size" curve: the same timing on views of one large buffer, NCCL alongside
    curve = []
    if args.curve:
        big_n = max(CURVE_BYTES) // esz
        big = ctx.empty(big_n, args.dtype)
        big.fill_(1.0)
        nbig = None if args.no_nccl else torch.ones(big_n, dtype=tdt, device=dev)
        tiny = torch.zeros(1, device=dev)
        for nbytes_c in CURVE_BYTES:
            view = big[:nbytes_c // esz]
            timed(ctx, lambda v=view: ctx.collective("allreduce", v), 3, lambda: flush_l2(scratch))
            ms = timed(ctx, lambda v=view: ctx.collective("allreduce", v), 10, lambda: flush_l2(scratch))
            us = statistics.median(ms) * 1e3
            pt = {"bytes": nbytes_c, "us": round(us, 2), "busbw_gbs": round(busbw(world, nbytes_c, us / 1e6), 2)}
            if nbig is not None:
                nv = nbig[:nbytes_c // esz]
                nt = []
                for it in range(13):
                    flush_l2(scratch)
                    dist.all_reduce(tiny)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record(stream)
                    dist.all_reduce(nv)
                    e.record(stream)
                    torch.cuda.synchronize()
                    if it >= 3:
                        nt.append(s.elapsed_time(e))
                nus = statistics.median(max_over_ranks(nt)) * 1e3
                pt["nccl_us"] = round(nus, 2)
                pt["nccl_busbw_gbs"] = round(busbw(world, nbytes_c, nus / 1e6), 2)
            curve.append(pt)
        del big, nbig

    # the reference's other two collectives on the same buffer (runtime.py:278-292):
    # busbw = (N-1)/N * S / t each (NCCL convention for reduce-scatter / all-gather)
    parts = {}
    for op in ("reduce_scatter", "allgather"):
        timed(ctx, lambda o=op: ctx.collective(o, work), 3, restore)
        ms = timed(ctx, lambda o=op: ctx.collective(o, work), 10, restore)
        us = statistics.median(ms) * 1e3
        parts[op] = {"us": round(us, 2), "busbw_gbs": round((world - 1) / world * nbytes / (us / 1e6) / 1e9, 2)}

    nccl = None
    if not args.no_nccl:
        nbuf = pristine.clone()
        tiny = torch.zeros(1, device=dev)
        for _ in range(3):
            dist.all_reduce(nbuf)
        torch.cuda.synchronize()
        nt = []
        for _ in range(10):
            nbuf.copy_(pristine)
            flush_l2(scratch)  # ends with a device spin: the host runs ahead
            dist.all_reduce(tiny)  # device-side alignment of the ranks, like ctx.barrier() on our arm
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            dist.all_reduce(nbuf)
            e.record(stream)
            torch.cuda.synchronize()
            nt.append(s.elapsed_time(e))
        nccl = round(busbw(world, nbytes, statistics.median(max_over_ranks(nt)) / 1e3), 2)

    # the reference's CPU multi-ring allreduce on this box's host cores, same job, same run
    # (rank 0; the other ranks wait at the barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        times, r_ = cpu_port_run(dims, n, budget_s=10.0)
        tc = statistics.median(times)
        cores = len(os.sched_getaffinity(0))
        cpu = {"value": round(busbw(world, n * 4, tc), 4), "unit": "GB/s", "cores": min(world, cores), "kind": "port",
               "sample": f"{len(times)} full allreduces of {n} fp32 x {world} ranks (grid {'x'.join(map(str, dims))}) "
                         f"with the C port of the reference runtime, one thread per rank; median {tc * 1e3:.1f} ms; "
                         f"host has {cores} cores"}
    dist.barrier()

    traffic_key = {2: "nvlink_tx_2_25.6M_f32", 4: "nvlink_tx_2x2_25.6M_f32"}.get(world)
    traffic = ncu_traffic(traffic_key) if (traffic_key and n == N_ELEM and args.dtype == "f32") else None
    if rank == 0:
        # peak: the recipe's measured NVLink figure (B200_PROFILING.md: 770 GB/s peer copy per direction).
        # The copy-engine ceiling measured in this run is reported beside it, not used: with more than
        # two GPUs the copy engines deliver LESS than this kernel.
        peak = MEASURED_PEER_GBS
        peak_src = ("B200_PROFILING.md measured peer copy per direction (770); the SM-issued payload ceiling with "
                    "both directions busy is ~700-706 on this box (DESIGN.md 5.3: probes + ncu protocol bytes)")
        line = {
            "metric": "multi-ring allreduce bus GB/s vs msg size at 2/4/8 B200; % of 900 GB/s NVLink",
            "value": round(bw, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (reference generate_input, seed 0)",
            "config": {"workload": workload_name(n, args.dtype, world, dims),
                       "placement": (f"{world} ranks sharing {ngpu} GPUs (functional check only: timings are "
                                     "not a measurement)") if shared else f"{world} GPUs, one rank each",
                       "ranks": world, "dims": list(dims), "bytes_per_rank": nbytes, "mode": args.mode,
                       "l2": "flushed between steps (256 MiB write per rank)",
                       "value_definition": "per-GPU busbw = 2(N-1)/N*S/t (NCCL convention), t = max over ranks"},
            "busbw_gbs": round(bw, 3), "aggregate_busbw_gbs": round(bw * world, 3),
            "pct_of_900": round(100 * bw / NOMINAL_NVLINK_GBS, 2), "algbw_gbs": round(nbytes / t / 1e9, 3),
            "other_grids": other or None,
            "graph_replay": graph_replay,
            "roofline": {"bound": "nvlink", "achieved": round(bw, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(bw / peak, 4), "traffic": traffic,
                         "traffic_kind": "NVLink TX bytes per launch per GPU (ncu nvltx__bytes.sum, user + protocol; "
                                         f"{world}-GPU harness, profiles/ncu_traffic.json)" if traffic else None,
                         "peak_source": peak_src, "ceiling": ceiling,
                         "frac_of_770": round(bw / MEASURED_PEER_GBS, 4), "frac_of_900": round(bw / NOMINAL_NVLINK_GBS, 4),
                         "algorithmic_bytes_per_launch": int(2 * (world - 1) / world * nbytes)},
            "nccl_busbw_gbs": nccl,
            "curve": curve or None,
            "reduce_scatter": parts["reduce_scatter"], "allgather": parts["allgather"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "step_ms": [round(x, 4) for x in step_ms],
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    dist.destroy_process_group()


def self_launch_command(argv, gpus: int, port: int) -> list:
    """`python bench.py --gpus N` without torchrun: one rank per GPU through
    torch.distributed.run, the same argv (the reference's launch() likewise
    spawns its own N workers, runtime.py:435-589)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(args) -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = {**os.environ, "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS", "1")}
    return subprocess.call(self_launch_command(sys.argv[1:], args.gpus, port), env=env)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        main_multi(args)
    elif args.gpus > 1:
        sys.exit(self_launch(args))
    else:
        main_single(args)


if __name__ == "__main__":
    main()
