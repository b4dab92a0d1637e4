"""Host-link rate of page-locked numpy memory (cudaHostRegister of a malloc'd
array) vs torch's pinned allocator (cudaHostAlloc), both directions at once
(diagnostic).  python tools/hostmem_probe.py [--mb 102.4] [--bufs 8]"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=102.4)
    ap.add_argument("--bufs", type=int, default=8)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_1708_02188_b200.hoststage import pin_array

    dev = torch.device("cuda", 0)
    n = int(args.mb * 1e6 / 4)
    devs = [torch.empty(n, device=dev) for _ in range(args.bufs)]
    devs2 = [torch.empty(n, device=dev) for _ in range(args.bufs)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def run(hin, hout, iters=6):
        ts = []
        for _ in range(iters):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(cur)
            s_in.wait_event(s)
            s_out.wait_event(s)
            with torch.cuda.stream(s_in):
                for h, d in zip(hin, devs):
                    d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s_out):
                for h, d in zip(hout, devs2):
                    h.copy_(d, non_blocking=True)
            cur.wait_stream(s_in)
            cur.wait_stream(s_out)
            e.record(cur)
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return statistics.median(ts[1:])

    pin_in = [torch.empty(n).pin_memory() for _ in range(args.bufs)]
    pin_out = [torch.empty(n).pin_memory() for _ in range(args.bufs)]
    np_in = [np.ones(n, dtype=np.float32) for _ in range(args.bufs)]
    np_out = [np.ones(n, dtype=np.float32) for _ in range(args.bufs)]
    for a in np_in + np_out:
        pin_array(a)
    reg_in = [torch.from_numpy(a) for a in np_in]
    reg_out = [torch.from_numpy(a) for a in np_out]
    t_pin = run(pin_in, pin_out)
    t_reg = run(reg_in, reg_out)
    gb = args.bufs * n * 4 / 1e9
    print(json.dumps({"probe": "host memory kind, H2D and D2H at once", "bufs": args.bufs, "mb_each": args.mb,
                      "torch_pinned_ms": round(t_pin, 3), "numpy_registered_ms": round(t_reg, 3),
                      "torch_pinned_gbs_each_way": round(gb / t_pin * 1e3, 1),
                      "numpy_registered_gbs_each_way": round(gb / t_reg * 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
