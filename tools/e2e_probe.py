"""Where does the N=1 e2e step lose time against the host link?  (diagnostic)

  python tools/e2e_probe.py [--ranks 8] [--n 25600000]

One GPU, `ranks` page-locked host arrays (runtime.host_empty) of n fp32, the
same bytes as bench.py's N=1 e2e leg.  Prints one JSON line per measurement
(median ms of --iters):
  link_bidi     H2D and D2H of every array at once on two streams (bench.py host_link_ms)
  h2d / d2h     one direction alone, one stream
  h2d_2s        one direction alone, arrays split over two streams
  copy_pipe     HostPipeline(lanes) with a no-op reduce: the copies' window structure alone
  pipe          HostPipeline(lanes) with the local-reduce kernel per window
  e2e           VirtualRanks.allreduce_host (the bench's e2e call, its default pipeline)
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
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--n", type=int, default=25_600_000)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--windows", default="2,3,4,6,8,12,16")
    ap.add_argument("--lanes", default="1")
    ap.add_argument("--align", default="1,65536,2097152")
    args = ap.parse_args()
    import torch

    from paper_1708_02188_b200.hoststage import HostPipeline
    from paper_1708_02188_b200.runtime import host_empty
    from paper_1708_02188_b200.virtual import VirtualRanks

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    R, n = args.ranks, args.n
    arrays = [host_empty(n, "f32") for _ in range(R)]
    for r, a in enumerate(arrays):
        a[...] = r + 1.0
    hosts = [torch.from_numpy(a) for a in arrays]
    back = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(R)]
    devs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(R)]
    devs2 = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(R)]
    streams = [torch.cuda.Stream(dev) for _ in range(4)]
    nbytes = R * n * 4

    def timed(fn):
        ts = []
        for _ in range(args.iters + 1):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for x in streams:
                x.wait_event(s)
            fn()
            for x in streams:
                stream.wait_stream(x)
            e.record(stream)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return statistics.median(ts[1:])

    def emit(what, ms, **kw):
        print(json.dumps({"probe": "e2e", "what": what, "ranks": R, "bytes_each_way": nbytes, "ms": round(ms, 3),
                          "gbs_each_way": round(nbytes / ms / 1e6, 2), **kw}), flush=True)

    def link_bidi():
        with torch.cuda.stream(streams[0]):
            for h, d in zip(hosts, devs2):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(streams[1]):
            for d, b in zip(devs, back):
                b.copy_(d, non_blocking=True)

    def h2d(k):
        def f():
            for i, (h, d) in enumerate(zip(hosts, devs)):
                with torch.cuda.stream(streams[i % k]):
                    d.copy_(h, non_blocking=True)
        return f

    def d2h(k):
        def f():
            for i, (d, b) in enumerate(zip(devs, back)):
                with torch.cuda.stream(streams[i % k]):
                    b.copy_(d, non_blocking=True)
        return f

    emit("link_bidi", timed(link_bidi))
    emit("h2d", timed(h2d(1)))
    emit("d2h", timed(d2h(1)))
    emit("h2d_2s", timed(h2d(2)))
    emit("d2h_2s", timed(d2h(2)))

    pairs = list(zip(arrays, devs))
    vr = VirtualRanks((2, 2, 2) if R == 8 else (R,), device=0, nblocks_per_rank=0) if R > 1 else None
    red = lambda lo, hi, s: vr.collective(devs, mode="local", stream=s, window=(lo, hi))  # noqa: E731
    for lanes in [int(x) for x in args.lanes.split(",")]:
        pipe = HostPipeline(dev, lanes=lanes)
        for w in [int(x) for x in args.windows.split(",")]:
            for taper in (True, False):
                for al in [int(x) for x in args.align.split(",")]:
                    if taper and w < 6:
                        continue
                    emit("copy_pipe", timed(lambda: pipe.run(pairs, n, w, lambda lo, hi, s: None, taper=taper,
                                                             align_bytes=al)),
                         windows=w, lanes=lanes, taper=taper, align_bytes=al)
                    if vr:
                        emit("pipe", timed(lambda: pipe.run(pairs, n, w, red, taper=taper, align_bytes=al)),
                             windows=w, lanes=lanes, taper=taper, align_bytes=al)
    if vr:
        for w in (4, 8):
            emit("e2e", timed(lambda: vr.allreduce_host(arrays, mode="local", windows=w)), windows=w)
        vr.close()


if __name__ == "__main__":
    main()
