"""Run one BASELINE config's solve a few times on cuda:0 (the command ncu profiles for
configs other than the C3 headline; tools/profile_c3.py is the C3 one):
    python tools/profile_cfg.py C4 [reps] [L]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from paper_2510_09204_b200 import solver  # noqa: E402
from sweep import workload  # noqa: E402

CONFIGS = {"C1": (4, 0, 1.0, 1, 1), "C2": (16, 10, 1.0, 32, 1), "C3": (32, 20, 2.0, 64, 8),
           "C4": (64, 30, 2.0, 128, 1), "C5n64": (64, 20, 2.83, 1024, 1), "C5n128": (128, 20, 4.0, 1024, 1)}


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 500
    n, m, h, inst, samp = CONFIGS[name]
    systems, xi, mi = workload(n, m, h, inst, samp, 1000 * int(name[1]))
    batch = solver.DeviceBatch(systems, xi, None, xi, cfg=solver.SolverConfig(max_iters=L),
                               member_instance=mi, early_exit=False, trace=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        batch.launch()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    print(name, batch.launch_info(), "ms per solve:",
          [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(reps)])


if __name__ == "__main__":
    main()
