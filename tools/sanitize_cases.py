"""Small launches for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool <tool> python tools/sanitize_cases.py [case ...]
cases: cluster8 (one C3 instance, 8 samples over 8-CTA clusters: the DSMEM / mbarrier
exchange), single (one member, one CTA), split (more members than resident CTAs: the split
schedule's cross-CTA handoff), big (n = 40 ring of FP32 hi/lo positions, 16-warp CTAs),
metrics (the epilogue kernels), vars (fixed_point_step's analysis kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2510_09204_b200 import solver  # noqa: E402
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble, build_basis,  # noqa: E402
                                           generate, sample_naive_prior, stack_xi)


def batch(n, m, inst, samples, h=2.0, seed=3000):
    basis = build_basis(BasisConfig(11, 100, 5.0))
    fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-h, h), n_obstacles=m)
    systems, xs = [], []
    for i in range(inst):
        scn = generate(fam, n, 2, seed=seed + i % 4, horizon=basis.config)
        systems.append(assemble(scn, basis))
        xs.append(solver.to_member_major(stack_xi(sample_naive_prior(scn, basis, samples, seed=seed + i)), n, 11))
    return systems, np.concatenate(xs), np.repeat(np.arange(inst), samples).astype(np.int32), basis


def run(case):
    if case == "cluster8":
        s, x, mi, _ = batch(32, 20, 1, 8)
        out = solver.solve_instances(s, x, None, x, member_instance=mi, cfg=solver.SolverConfig(max_iters=5),
                                     fixed_iterations=True, cluster=8)
    elif case == "single":
        s, x, mi, _ = batch(32, 20, 1, 1)
        out = solver.solve_instances(s, x, None, x, member_instance=mi, cfg=solver.SolverConfig(max_iters=5),
                                     fixed_iterations=True, cluster=1)
    elif case == "split":
        s, x, mi, _ = batch(32, 20, 75, 4)       # 300 members > 296 resident CTAs
        out = solver.solve_instances(s, x, None, x, member_instance=mi, cfg=solver.SolverConfig(max_iters=3),
                                     fixed_iterations=True, cluster=1)
    elif case == "big":
        s, x, mi, _ = batch(40, 12, 1, 2)
        out = solver.solve_instances(s, x, None, x, member_instance=mi, cfg=solver.SolverConfig(max_iters=3),
                                     fixed_iterations=True, cluster=1)
    elif case == "metrics":
        from paper_2510_09204_b200 import metrics
        s, x, mi, basis = batch(8, 3, 1, 2)
        solver.kinematic_peaks(x, basis)
        out = None
        metrics.metrics_batch(x, basis, [])
    elif case == "vars":
        s, x, mi, _ = batch(6, 2, 1, 2)
        xr = np.moveaxis(x.reshape(2, 2, -1), 0, -1)
        solver.fixed_point_step(solver.SolverState(xi=xr, lam=np.zeros_like(xr)), s[0],
                                solver.ObjectiveMode.projection(xr), solver.SolverConfig())
        out = None
    else:
        raise SystemExit(f"unknown case {case}")
    if out is not None:
        assert np.all(np.isfinite(out.xi)), case
    print(f"{case}: ok", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or ["cluster8", "single", "split", "big", "metrics", "vars"]:
        run(c)
