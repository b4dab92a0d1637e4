"""Profilable NVLink view of the allreduce kernel (single process, 2 GPUs).

ncu must not wrap the multi-rank run (replaying a kernel that waits on a peer's
flags would hang), so this harness runs the SAME rbx_step_kernel<float> with a
flag-free plan: grid (2,), rank 0's buffer on cuda:0, rank 1's on cuda:1 (peer
access enabled), one launch on cuda:0 folding both owned regions.  GPU 0 then
reads rank 1's whole buffer over NVLink and writes the result back into it:
S bytes in each direction, the same 16-byte load/fold/store loop as the
multi-GPU FUSED mode.  ncu's Nvlink section reports the bytes and % of peak.

  python tools/nvlink_ncu.py [--elems 25600000] [--iters 20]
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=25_600_000)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch

    from paper_1708_02188_b200.runtime import Workload, generate_input
    from paper_1708_02188_b200.virtual import VirtualRanks

    n = args.elems
    wl = Workload(lengths=(n,), dtype="f32", seed=0)
    parts = [generate_input(wl, 0, r, n) for r in range(2)]
    bufs = [torch.from_numpy(parts[0]).to("cuda:0"), torch.from_numpy(parts[1]).to("cuda:1")]
    vr = VirtualRanks((2,), device=0, peer_devices=(1,))
    torch.cuda.set_device(0)
    vr.collective(bufs, mode="local")
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    # grid (2,): every element is x0 + x1 (one IEEE add, commutative), so torch's
    # add is the reference order here
    want = torch.from_numpy(parts[0]) + torch.from_numpy(parts[1])
    ok = all(torch.equal(b.cpu(), want) for b in bufs)
    stream = torch.cuda.current_stream(0)
    ts = []
    for _ in range(args.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        vr.collective(bufs, mode="local")
        e.record(stream)
        torch.cuda.synchronize(0)
        ts.append(s.elapsed_time(e) / 1e3)
    t = statistics.median(ts)
    S = n * 4
    print(json.dumps({"harness": "grid (2,), one launch on cuda:0, rank-1 buffer on cuda:1 over NVLink",
                      "bit_exact_vs_reference_order": ok, "elems": n, "kernel_us": round(t * 1e6, 1),
                      "nvlink_bytes_each_direction": S, "achieved_gbs_each_direction": round(S / t / 1e9, 1),
                      "pct_of_900": round(100 * S / t / 1e9 / 900, 1)}), flush=True)


if __name__ == "__main__":
    main()
