"""Copy-engine NVLink probe: peer memcpy throughput, one process, 2+ GPUs.

  python tools/ce_probe.py [--mb 51.2] [--streams 1,2,4,8]

Cases per stream count k (the buffer split into k pieces, one stream each):
  push_1dir  gpu0 -> gpu1, copies issued on gpu0's streams
  pull_1dir  gpu0 -> gpu1, copies issued on gpu1's streams
  push_bidi  gpu0 -> gpu1 and gpu1 -> gpu0 at once (each on its source GPU)
  pull_bidi  both directions, each issued on the destination GPU
GB/s per direction = bytes / time (CUDA events around all copies, after a
cross-device join).  Compare with tools/nvlink_probe.cu (SM loads/stores).
"""

from __future__ import annotations

import argparse
import json
import statistics

import torch


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--mb", type=float, default=51.2)
    p.add_argument("--streams", default="1,2,4,8")
    p.add_argument("--iters", type=int, default=10)
    a = p.parse_args()
    assert torch.cuda.device_count() >= 2
    n = int(a.mb * 1e6) // 4
    bufs = {}
    for d in (0, 1):
        with torch.cuda.device(d):
            bufs[d] = (torch.randn(n, device=f"cuda:{d}"), torch.empty(n, device=f"cuda:{d}"))
    for d in (0, 1):
        assert torch.cuda.can_device_access_peer(d, 1 - d)
    # warm up peer mappings (torch enables peer access lazily on first copy)
    bufs[1][1].copy_(bufs[0][0])
    bufs[0][1].copy_(bufs[1][0])
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    streams = {d: [torch.cuda.Stream(device=d) for _ in range(8)] for d in (0, 1)}

    def run(kind, k):
        times = []
        for _ in range(a.iters + 2):
            for d in (0, 1):
                torch.cuda.synchronize(d)
            s0 = torch.cuda.Event(enable_timing=True)
            e0 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(0):
                torch.cuda._sleep(20_000)
                s0.record()
            with torch.cuda.device(1):
                torch.cuda.current_stream(1).wait_event(s0)
            dirs = [(0, 1)] if kind.endswith("1dir") else [(0, 1), (1, 0)]
            done = []
            for src, dst in dirs:
                issuer = src if kind.startswith("push") else dst
                for i in range(k):
                    lo, hi = n * i // k, n * (i + 1) // k
                    st = streams[issuer][i]
                    st.wait_event(s0)
                    with torch.cuda.stream(st):
                        bufs[dst][1][lo:hi].copy_(bufs[src][0][lo:hi], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(st)
                    done.append(ev)
            with torch.cuda.device(0):
                cs = torch.cuda.current_stream(0)
                for ev in done:
                    cs.wait_event(ev)
                e0.record()
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            times.append(s0.elapsed_time(e0))
        ms = statistics.median(times[2:])
        return ms

    for k in [int(x) for x in a.streams.split(",")]:
        for kind in ("push_1dir", "pull_1dir", "push_bidi", "pull_bidi"):
            ms = run(kind, k)
            print(json.dumps({"case": kind, "streams": k, "bytes": n * 4, "ms": round(ms, 4),
                              "gbs_per_dir": round(n * 4 / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
