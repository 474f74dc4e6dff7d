"""Run the C3 headline solve (rank-0 batch: 64 instances x 8 samples, L=500) a few
times on cuda:0 — the command profiled by ncu (profiles/README.md)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    L = int(sys.argv[2]) if len(sys.argv) > 2 else bench.WL["L"]
    systems, xi, mi = bench.make_workload(0)
    cfg = solver.SolverConfig(max_iters=L)
    batch = solver.DeviceBatch(systems, xi, None, xi, cfg=cfg, member_instance=mi,
                               early_exit=False, trace=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        batch.launch()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    print("ms per solve:", [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(reps)])


if __name__ == "__main__":
    main()
