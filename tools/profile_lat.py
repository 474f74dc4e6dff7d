"""Run the latency case (one C3 instance = 8 members, L=500, 8-CTA clusters) a few times on
cuda:0 — the command profiled by ncu for the latency path (profiles/README.md)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cluster = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    systems, xi, mi = bench.make_workload(0)
    cfg = solver.SolverConfig(max_iters=bench.WL["L"])
    batch = solver.DeviceBatch([systems[0]], xi[:8], None, xi[:8], cfg=cfg, early_exit=False,
                               trace=True, cluster=cluster)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        batch.launch()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    print("ms per solve:", [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(reps)])


if __name__ == "__main__":
    main()
