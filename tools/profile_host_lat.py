"""Host-side cost of the latency path (one C3 instance = 8 members, L = 500, host arrays in
and out through solve_instances): p50 of the whole call and of its phases (system extraction,
input packing + H2D, kernel, D2H + unpacking) over distinct scenarios, then a cProfile of the
Python side. Run on the GPU box: python tools/profile_host_lat.py [n_scenarios]"""
import cProfile
import os
import pstats
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    S = bench.WL["samples"]
    cfg = solver.SolverConfig(max_iters=bench.WL["L"])
    lsys, lxi, _ = bench.make_workload(bench.LAT_SEED_RANK, dict(bench.WL, instances=N))
    solver.solve_instances([lsys[0]], lxi[:S], None, lxi[:S], cfg=cfg, fixed_iterations=True)
    ph = {k: [] for k in ("total", "system", "batch", "kernel", "results")}
    for i in range(N):
        sel = slice(i * S, (i + 1) * S)
        t0 = time.perf_counter()
        solver.system_data(lsys[i], "projection", cfg.rho)
        t1 = time.perf_counter()
        b = solver.DeviceBatch([lsys[i]], lxi[sel], None, lxi[sel], cfg=cfg, early_exit=False)
        t2 = time.perf_counter()
        b.launch()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        b.results()
        t4 = time.perf_counter()
        for k, v in zip(ph, (t4 - t0, t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            ph[k].append(1e3 * v)
    print("phases, p50 ms over %d distinct scenarios (system memoised after its first use):" % N)
    for k, v in ph.items():
        print(f"  {k:8s} {statistics.median(v):7.3f}")
    # whole call, fresh scenarios (the bench's latency protocol)
    lsys2, lxi2, _ = bench.make_workload(bench.LAT_SEED_RANK + 1, dict(bench.WL, instances=N))
    pr = cProfile.Profile()
    tt = []
    for i in range(N):
        sel = slice(i * S, (i + 1) * S)
        t0 = time.perf_counter()
        pr.enable()
        solver.solve_instances([lsys2[i]], lxi2[sel], None, lxi2[sel], cfg=cfg,
                               fixed_iterations=True, trace=True)
        pr.disable()
        tt.append(1e3 * (time.perf_counter() - t0))
    print("solve_instances p50 %.3f ms (under cProfile)" % statistics.median(tt))
    pstats.Stats(pr).sort_stats("tottime").print_stats(20)


if __name__ == "__main__":
    main()
