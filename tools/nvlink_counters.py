"""NVLink traffic evidence without a profiler: NVML NVLink throughput counters
(data payload TX/RX bytes) read before and after K allreduces on every rank.

  torchrun --nproc-per-node N tools/nvlink_counters.py [--elems 25600000] [--iters 50]

Prints per-rank measured NVLink data bytes per allreduce next to the
algorithmic bus bytes 2(N-1)/N*S, plus the implied achieved GB/s per
direction (bytes / kernel time).  ncu cannot wrap a multi-rank run (kernel
replay of flag-synchronised kernels), so this is the NVLink-side evidence.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def nvml_counters(handle, pynvml, kind="DATA"):
    """(tx_bytes, rx_bytes) summed over links, from NVML field values (KiB units).
    kind DATA: payload only; RAW: payload + protocol (headers, read requests, acks)."""
    fids = []
    for name in (f"NVML_FI_DEV_NVLINK_THROUGHPUT_{kind}_TX", f"NVML_FI_DEV_NVLINK_THROUGHPUT_{kind}_RX"):
        fids.append(getattr(pynvml, name, None))
    if None in fids:
        return None
    out = []
    for fid in fids:
        total, seen = 0, 0
        for link in range(18):  # NVLink 5: 18 links per GPU
            try:
                (v,) = pynvml.nvmlDeviceGetFieldValues(handle, [(fid, link)])
            except Exception:
                continue
            if v.nvmlReturn == 0:
                total += int(v.value.ullVal)
                seen += 1
        if not seen:
            return None
        out.append(total * 1024)  # counters are in KiB
    return tuple(out)


def smi_counters(index: int):
    """Fallback: `nvidia-smi nvlink -gt d` per-link Data Tx/Rx counters (KiB)."""
    import re
    import subprocess

    try:
        txt = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True, text=True,
                             timeout=30).stdout
    except Exception:
        return None, ""
    tx = rx = 0
    seen = False
    for line in txt.splitlines():
        m = re.search(r"Data (Tx|Rx):\s*([0-9]+)\s*KiB", line)
        if m:
            seen = True
            if m.group(1) == "Tx":
                tx += int(m.group(2)) * 1024
            else:
                rx += int(m.group(2)) * 1024
    return ((tx, rx) if seen else None), txt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=25_600_000)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--mode", default="auto")
    args = ap.parse_args()
    import pynvml
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(rank)
    dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}.get(world, (world,))
    ctx = RankContext(rank, Grid(dims), device=rank, blocking=False)
    work = ctx.empty(args.elems, "f32")
    work.normal_()
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        ctx.collective("allreduce", work, mode=args.mode)
        work.mul_(1.0 / world)
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(0.5)
    c0 = nvml_counters(h, pynvml)
    r0 = nvml_counters(h, pynvml, "RAW")
    src = "nvml"
    raw0 = ""
    if c0 is None:
        c0, raw0 = smi_counters(rank)
        src = "nvidia-smi nvlink -gt d"
    ts = []
    for _ in range(args.iters):
        ctx.barrier()  # align ranks so kernel_us is the collective, not the skew
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.collective("allreduce", work, mode=args.mode)
        e.record(stream)
        work.mul_(1.0 / world)  # local, no NVLink traffic
        ts.append((s, e))
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(0.5)
    c1 = nvml_counters(h, pynvml) if src == "nvml" else smi_counters(rank)[0]
    r1 = nvml_counters(h, pynvml, "RAW") if src == "nvml" else None
    kt = sum(s.elapsed_time(e) for s, e in ts) / len(ts) / 1e3
    S = args.elems * 4
    alg = 2 * (world - 1) / world * S
    row = {"rank": rank, "n_gpus": world, "dims": list(dims), "bytes_per_rank": S, "mode": args.mode,
           "algorithmic_bus_bytes_per_direction": alg, "kernel_us": round(kt * 1e6, 1)}
    if c0 and c1:
        tx = (c1[0] - c0[0]) / args.iters
        rx = (c1[1] - c0[1]) / args.iters
        row.update({"nvlink_tx_bytes_per_allreduce": tx, "nvlink_rx_bytes_per_allreduce": rx,
                    "tx_over_alg": round(tx / alg, 4), "rx_over_alg": round(rx / alg, 4),
                    "achieved_tx_gbs": round(tx / kt / 1e9, 1), "achieved_rx_gbs": round(rx / kt / 1e9, 1)})
        if r0 and r1:
            rtx = (r1[0] - r0[0]) / args.iters
            rrx = (r1[1] - r0[1]) / args.iters
            row.update({"nvlink_raw_tx_bytes_per_allreduce": rtx, "nvlink_raw_rx_bytes_per_allreduce": rrx,
                        "raw_over_data_tx": round(rtx / tx, 4) if tx else None,
                        "raw_over_data_rx": round(rrx / rx, 4) if rx else None,
                        "raw_tx_gbs": round(rtx / kt / 1e9, 1), "raw_rx_gbs": round(rrx / kt / 1e9, 1)})
    else:
        row["nvml"] = "NVLink throughput fields unavailable"
        row["smi_raw_head"] = raw0[:600]
    row["counter_source"] = src
    rows = [None] * world
    dist.all_gather_object(rows, row)
    if rank == 0:
        for r in rows:
            print(json.dumps(r), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
