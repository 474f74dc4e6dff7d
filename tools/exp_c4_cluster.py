"""n > 32 experiment: device time of the L=500 solve for n=64 (30 obstacles) over batch size
and cluster size (the auto cluster policy of sfb_solve is set from these numbers)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep import workload  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = int(sys.argv[2]) if len(sys.argv) > 2 else 30
insts = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [32, 64, 128, 256, 512]
for inst in insts:
    systems, xi, mi = workload(n, m, max(1.0, 2.0 * (n / 32) ** 0.5) if n != 64 else 2.0, inst, 1, 7000)
    row = []
    for cl in (0, 1, 2, 4, 8):
        b = solver.DeviceBatch(systems, xi, None, xi, cfg=solver.SolverConfig(max_iters=500),
                               member_instance=mi, early_exit=False, trace=False, cluster=cl)
        b.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.launch()
        e1.record()
        torch.cuda.synchronize()
        row.append(f"c={cl or 'auto'}: {e0.elapsed_time(e1):7.2f} ms")
    print(f"n={n} m={m} I={inst:4d}  " + "  ".join(row), flush=True)
