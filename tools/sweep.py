"""Throughput of the SF kernel across the BASELINE.json configs (C1-C4) and the
robots x batch sweep (C5: 8-128 robots, batch 1-1024 instances, 20 obstacles,
box half-width max(1, 2 sqrt(n/32)), T=100, L=500). Device-timed
(CUDA events, inputs resident), one GPU. Every row carries the roofline fraction of
the SURVEY §8(d) screened model (FP32 flops with the kernel's own active-row count,
against profiles/peaks_b200.json); with --cpu the named configs also get the CPU
reference (oracle/sf_dense.py port, bench.CpuReference: one synchronized instance per
host core; C1 run in full, C2-C4 over L_cpu = 5 evaluations, extrapolated) and the
GPU/CPU ratio.

    python tools/sweep.py [--quick] [--cpu] [--out=<file name under profiles/>]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

from paper_2510_09204_b200 import solver  # noqa: E402
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble, build_basis,  # noqa: E402
                                           generate, sample_naive_prior, stack_xi)


def workload(n, m, h, instances, samples, seed0):
    basis = build_basis(BasisConfig(11, 100, 5.0))
    fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-h, h), n_obstacles=m)
    systems, xs = [], []
    uniq = min(instances, 64)   # distinct scenarios (generation is host-side and slow at n=128)
    for i in range(uniq):
        scn = generate(fam, n, 2, seed=seed0 + i, horizon=basis.config)
        systems.append(assemble(scn, basis))
        xs.append(solver.to_member_major(stack_xi(sample_naive_prior(scn, basis, samples, seed=seed0 + i)), n, 11))
    reps = [i % uniq for i in range(instances)]
    xi = np.concatenate([xs[r] for r in reps])
    mi = np.repeat(np.arange(instances), samples).astype(np.int32)
    return [systems[r] for r in reps], xi, mi


def roofline_frac(systems, xi, mi, L, seconds, n, m):
    """FP32 model flops of one solve (bench.algorithmic_ops, active rows counted by the kernel)
    over its time, as a fraction of the measured FFMA2 peak."""
    cfg = solver.SolverConfig(max_iters=L)
    b = solver.DeviceBatch(systems, xi, None, xi, cfg=cfg, member_instance=mi, early_exit=False,
                           trace=False, counters=True)
    b.launch()
    c = b.out_counters.cpu().numpy()
    o32, _ = bench.algorithmic_ops(n, m, 100, 11, 2, 6, int(c[:, 1].sum()), int(c[:, 3].sum()))
    peaks, _ = bench.load_peaks()
    return o32 / seconds / 1e12 / peaks["fp32_ffma2_tflops"]


def cpu_row(name, n, m, h, inst, samp, L):
    """CPU reference instances/s for a named config (seeds as the GPU rows)."""
    wl = dict(bench.WL, name=name, n=n, m=m, h=h, samples=samp, L=L)
    full = name == "C1"                          # C1 runs in full
    ref = bench.CpuReference(L_cpu=L if full else 5, steps=1, warmup=0 if full else 1, wl=wl,
                             seed0=1000 * int(name[1]))
    try:
        vals = ref.run()
    finally:
        ref.close()
    d = ref.describe(vals)
    return {"cpu_instances_per_s": d["median"], "cpu_cores": d["cores"], "cpu_model": d["cpu_model"],
            "cpu_L": ref.L, "cpu_extrapolated": not full, "cpu_setup_s": d["setup_s_per_instance"]}


def time_solve(systems, xi, mi, L, reps=3):
    cfg = solver.SolverConfig(max_iters=L)
    batch = solver.DeviceBatch(systems, xi, None, xi, cfg=cfg, member_instance=mi, early_exit=False,
                               trace=False)
    batch.launch()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        ev[0].record()
        batch.launch()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
    return min(ts), batch.plan.smem_bytes


def main():
    quick = "--quick" in sys.argv
    with_cpu = "--cpu" in sys.argv
    out = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")), "r02_sweep.json")
    L = 500
    rows = []
    named = [("C1", 4, 0, 1.0, 1, 1), ("C2", 16, 10, 1.0, 32, 1), ("C3", 32, 20, 2.0, 64, 8),
             ("C4", 64, 30, 2.0, 128, 1)]
    for name, n, m, h, inst, samp in named:
        systems, xi, mi = workload(n, m, h, inst, samp, 1000 * int(name[1]))
        t, smem = time_solve(systems, xi, mi, L)
        rows.append(dict(config=name, robots=n, obstacles=m, instances=inst, samples=samp,
                         members=inst * samp, L=L, seconds=t, instances_per_s=inst / t,
                         member_iters_per_s=inst * samp * (L + 1) / t, smem_bytes=smem,
                         fp32_roofline_frac=roofline_frac(systems, xi, mi, L, t, n, m)))
        if with_cpu:
            rows[-1].update(cpu_row(name, n, m, h, inst, samp, L))
            rows[-1]["gpu_over_cpu"] = rows[-1]["instances_per_s"] / rows[-1]["cpu_instances_per_s"]
        print(json.dumps(rows[-1]), flush=True)
    robots = [8, 16, 32, 64, 128]
    batches = [1, 8, 64, 256, 1024] if not quick else [1, 64]
    for n in robots:
        h = max(1.0, 2.0 * math.sqrt(n / 32))
        for inst in batches:
            systems, xi, mi = workload(n, 20, h, inst, 1, 5000 + n)
            t, smem = time_solve(systems, xi, mi, L, reps=2)
            rows.append(dict(config="C5", robots=n, obstacles=20, instances=inst, samples=1,
                             members=inst, L=L, seconds=t, instances_per_s=inst / t,
                             member_iters_per_s=inst * (L + 1) / t, smem_bytes=smem,
                             fp32_roofline_frac=roofline_frac(systems, xi, mi, L, t, n, 20)))
            print(json.dumps(rows[-1]), flush=True)
    with open(os.path.join(ROOT, "profiles", out), "w") as fh:
        json.dump({"gpu": torch.cuda.get_device_name(0), "rows": rows,
                   "note": "device-timed solve (CUDA events), inputs resident; C5 uses 20 obstacles, "
                           "box half-width max(1, 2 sqrt(n/32)), 1 sample, naive-prior warm start"},
                  fh, indent=1)


if __name__ == "__main__":
    main()
