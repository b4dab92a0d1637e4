"""Small single-GPU self-check of every kernel mode (race /
sync / memory checking).  Every mode of the multi-rank kernel runs as virtual
ranks of one cooperative launch (flags, epochs, pushes, dynamic tiles), plus
the local-reduce and LL kernels, on small ragged buffers, twice (epochs and
tile counters advanced), and every rank's bits are compared with the
reference-order fold.  Meant to run under compute-sanitizer
(memcheck / racecheck / synccheck / initcheck); on this sandbox's GPU pool the
sanitizer is closed (tools/gpurun/r72.sh shows the refusal), so it runs bare.

  [compute-sanitizer --tool memcheck] python tests/sanitize_workload.py [--modes local,fused,...]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="local,fused,ring_dims,fused_pull,push,ll")
    ap.add_argument("--length", type=int, default=200_011)  # > 2 tiles per CTA: dynamic tiles
    args = ap.parse_args()
    import numpy as np
    import torch

    from oracle import ringbox_oracle as orc
    from paper_1708_02188_b200.virtual import VirtualRanks

    for dims in ((2, 2), (2, 2, 2)):
        grid = orc.Grid(dims)
        n = grid.size
        parts = [orc.generate_input(3, 0, r, args.length, "f32") for r in range(n)]
        want = orc.closed_form_allreduce(grid, parts)
        for mode in args.modes.split(","):
            vr = VirtualRanks(dims, nblocks_per_rank=0 if mode == "local" else 2, timeout_s=120.0)
            for _ in range(2):  # second call: epochs advanced, dynamic-tile counters rewound
                ts = [torch.from_numpy(p.copy()).cuda() for p in parts]
                vr.collective(ts, mode=mode)
                torch.cuda.synchronize()
                vr.check()
                ok = all(np.array_equal(t.cpu().numpy(), want) for t in ts)
                print(f"dims={dims} mode={mode} bit_exact={ok}", flush=True)
                if not ok:
                    sys.exit(2)
            vr.close()


if __name__ == "__main__":
    main()
