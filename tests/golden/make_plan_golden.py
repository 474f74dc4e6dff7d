"""Golden vectors of the planner around the SF, made by running the REFERENCE's
`swarmplan.pipeline.plan` (pkg/src/swarmplan/pipeline.py:88-153).

    python tests/golden/make_plan_golden.py       # writes tests/golden/plan_*.npz

Each fixture holds the scenario (starts, goals, radii, box, obstacles as (n_obs, 3, 3)
center/velocity/radii, horizon), the candidates (C, n, n_d, n_basis), top_k and the
SolverConfig, and the reference's outputs: pre/post residuals, smoothness, order, the
chosen index and status, the chosen coefficients and the refined members' iterations.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from swarmplan.basis import BasisConfig, build_basis  # noqa: E402
from swarmplan.pipeline import plan, sample_naive_prior  # noqa: E402
from swarmplan.scenario import Obstacle, ScenarioFamily, generate  # noqa: E402
from swarmplan.solver import SolverConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _obs(scn):
    arr = np.zeros((len(scn.obstacles), 3, 3))
    for o, ob in enumerate(scn.obstacles):
        arr[o, 0, : len(ob.center)] = ob.center
        arr[o, 1, : len(ob.velocity)] = ob.velocity
        arr[o, 2, : len(ob.radii)] = ob.radii
    return arr


def save(name, scn, count, top_k, cfg, seed):
    basis = build_basis(scn.horizon)
    batch = sample_naive_prior(scn, basis, count, seed=seed)
    cands = np.stack(batch.candidates)
    res = plan(scn, batch, top_k=top_k, cfg=cfg, basis=basis)
    h = scn.horizon
    np.savez_compressed(
        os.path.join(OUT, f"plan_{name}.npz"),
        n=scn.n, n_d=scn.n_d, radii=scn.radii, starts=scn.starts, goals=scn.goals,
        p_min=scn.p_min, p_max=scn.p_max, obstacles=_obs(scn),
        horizon=np.array([h.n_basis, h.num_steps, h.duration]), candidates=cands, top_k=top_k,
        cfg=np.array([cfg.rho, cfg.max_iters, cfg.primal_tol, cfg.fp_tol, cfg.d_max]),
        pre=batch.pre_residual, post=batch.post_residual, smooth=batch.smoothness,
        order=res.order, index=res.index, status=res.status, coeffs=res.coeffs,
        iterations=np.array([r.iterations for r in res.refined]),
        statuses=np.array([r.status for r in res.refined]))
    print(name, res.status, res.index, [r.iterations for r in res.refined])


def main():
    hz = BasisConfig(11, 50, 5.0)
    scn = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=3), 8, 2, seed=41,
                   horizon=hz)
    # converging refinement (default tolerances, bounded iterations)
    save("obs8_default", scn, 12, 4, SolverConfig(max_iters=2000), 41)
    # too few iterations for any refined candidate to reach primal_tol -> infeasible_best_effort,
    # chosen by post residual (a 1e-300 tolerance would instead hit the documented exact-zero
    # difference)
    save("obs8_short", scn, 12, 4, SolverConfig(max_iters=15), 41)
    # 3D with a moving obstacle
    scn3 = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=2), 6, 3, seed=43,
                    horizon=hz)
    scn3.obstacles = [Obstacle(center=o.center, radii=o.radii, velocity=0.05 * np.ones(3) * (-1) ** k)
                      for k, o in enumerate(scn3.obstacles)]
    save("d3_default", scn3, 8, 3, SolverConfig(max_iters=2000), 43)


if __name__ == "__main__":
    main()
