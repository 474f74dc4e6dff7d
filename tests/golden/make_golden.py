"""Generate the golden vectors of the SF hot path by running the REFERENCE itself.

Run in the dev container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Each fixture holds the full input of one `swarmplan.solver.solve_batch` call
(pkg/src/swarmplan/solver.py:286) — the constraint-system arrays the solver
reads, the objective, the warm start and the config — plus the reference's
outputs: final xi / lambda per member, status, iterations, final primal, the
full (primal, fixed-point) trace and eq_violation_max. The GPU box has no
reference; the parity tests rebuild the call from these arrays.
"""

from __future__ import annotations

import os
import sys
import time

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from swarmplan.basis import BasisConfig, build_basis, straight_line_coeffs  # noqa: E402
from swarmplan.constraints import DEFAULT_MARGIN, assemble  # noqa: E402
from swarmplan.pipeline import sample_naive_prior  # noqa: E402
from swarmplan.scenario import Obstacle, Scenario, ScenarioFamily, generate  # noqa: E402
from swarmplan.solver import (  # noqa: E402
    ObjectiveMode, SolverConfig, SolverState, cold_start, fixed_point_step, solve_batch,
    stack_xi, state_from_xi, xi_from_coeffs,
)

OUT = os.path.dirname(os.path.abspath(__file__))
STATUS = {"max_iters": 0, "converged_primal": 1, "converged_fp": 2}
FIXED = dict(primal_tol=1e-300, fp_tol=1e-300)


def save(name, sys_, mode, state, cfg, results, note=""):
    d = sys_.dims
    B = state.xi.shape[-1]
    T = max(len(r.trace) for r in results)
    trace = np.full((B, T, 2), np.nan)
    for b, r in enumerate(results):
        trace[b, : len(r.trace)] = r.trace
    if mode.kind == "projection":
        t = np.asarray(mode.target, float)
        t = t[:, :, None] if t.ndim == 2 else t
    else:
        t = np.zeros((d.n_d, d.nvar_ax, 0))
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        dims=np.array([d.n, d.n_d, d.n_basis, d.num_steps, d.n_obs, d.a_rows, d.g_rows]),
        W=sys_.basis.W, Wd=sys_.basis.Wd, Wdd=sys_.basis.Wdd, grid=sys_.basis.grid,
        duration=sys_.basis.config.duration,
        A=sys_.A, b=sys_.b, h=sys_.h, pair_axes=sys_.pair_axes, obs_axes=sys_.obs_axes,
        obs_pos=sys_.obs_pos, d_max=sys_.d_max,
        kind=np.array(mode.kind), target=t,
        xi0=state.xi, lam0=state.lam,
        cfg=np.array([cfg.rho, cfg.max_iters, cfg.primal_tol, cfg.fp_tol, cfg.d_max]),
        out_xi=np.stack([r.xi for r in results]), out_lam=np.stack([r.lam for r in results]),
        out_status=np.array([STATUS[r.status] for r in results]),
        out_iterations=np.array([r.iterations for r in results]),
        out_primal=np.array([r.primal for r in results]),
        out_trace=trace, out_eq=np.array([r.eq_violation_max for r in results]),
        note=np.array(note),
    )
    its = [r.iterations for r in results]
    print(f"{name:22s} n={d.n:3d} m={d.n_obs:2d} nd={d.n_d} B={B:2d} iters={min(its)}..{max(its)} "
          f"status={sorted(set(r.status for r in results))} primal[0]={results[0].primal:.3e}")


WANT = set(sys.argv[1:])


def want(name):
    return not WANT or name in WANT


def run(name, scn, basis, xi, lam, kind, cfg, rest_to_rest=True, note=""):
    if not want(name):
        return 0.0
    sys_ = assemble(scn, basis, rest_to_rest=rest_to_rest, d_max=cfg.d_max)
    mode = ObjectiveMode.projection(xi) if kind == "projection" else ObjectiveMode.smoothness()
    st = SolverState(xi=xi, lam=lam)
    t0 = time.perf_counter()
    res = solve_batch(st, sys_, mode, cfg)
    save(name, sys_, mode, st, cfg, res, note)
    return time.perf_counter() - t0


def naive(scn, basis, count, seed, lam_scale=0.0, lam_seed=99):
    cands = sample_naive_prior(scn, basis, count=count, seed=seed).candidates
    xi = stack_xi(cands)
    lam = lam_scale * np.random.default_rng(lam_seed).standard_normal(xi.shape)
    return xi, lam


def swap(seed, horizon=None, radius=0.1):
    """tests/conftest.py:19-34 (two robots exchanging random positions)."""
    horizon = horizon or BasisConfig()
    rng = np.random.default_rng(seed)
    while True:
        starts = rng.uniform(-0.85, 0.85, size=(2, 2))
        if np.linalg.norm(starts[0] - starts[1]) > 4.0 * radius:
            break
    scn = Scenario(n=2, n_d=2, radii=[radius] * 3, starts=starts, goals=starts[::-1].copy(),
                   obstacles=[], p_min=[-1.0, -1.0], p_max=[1.0, 1.0], horizon=horizon, seed=seed)
    scn.validate()
    return scn


def main():
    b100 = BasisConfig(11, 100, 5.0)
    B100 = build_basis(b100)
    B50 = build_basis(BasisConfig())
    fam = lambda m, h: ScenarioFamily("random_box", robot_radius=0.1, box=(-h, h), n_obstacles=m)

    # C1: 4 robots, no obstacles, T=100, 1 member, fixed 500 iterations (BASELINE configs[0])
    scn = generate(fam(0, 1.0), 4, 2, seed=1001, horizon=b100)
    xi, lam = naive(scn, B100, 1, seed=1001)
    run("c1_fixed500", scn, B100, xi, lam, "projection", SolverConfig(max_iters=500, **FIXED),
        note="BASELINE configs[0]: 4 robots, T=100, 1x1, L=500 fixed")
    xi, lam = naive(scn, B100, 4, seed=7, lam_scale=0.3)
    run("c1_noisy_b4", scn, B100, xi, lam, "projection", SolverConfig(max_iters=200, **FIXED))

    # C2-like: 16 robots, 10 obstacles, [-1,1]^2 (heavily infeasible) and [-2,2]^2 (converging)
    scn = generate(fam(10, 1.0), 16, 2, seed=2001, horizon=b100)
    xi, lam = naive(scn, B100, 4, seed=2001)
    run("c2_infeasible_L60", scn, B100, xi, lam, "projection", SolverConfig(max_iters=60, **FIXED),
        note="16/10 in [-1,1]: the FP-drift stress case")
    scn = generate(fam(4, 2.0), 8, 2, seed=2002, horizon=B50.config)
    xi, lam = naive(scn, B50, 3, seed=2002)
    run("conv8_default_tol", scn, B50, xi, lam, "projection", SolverConfig(max_iters=3000),
        note="default tolerances; convergence-mode status/iterations parity")

    # C3 / C4 shapes, short fixed runs (headline workload shapes)
    scn = generate(fam(20, 2.0), 32, 2, seed=3000, horizon=b100)
    xi, lam = naive(scn, B100, 8, seed=3000)
    run("c3_inst0_L4", scn, B100, xi, lam, "projection", SolverConfig(max_iters=4, **FIXED),
        note="BASELINE configs[2] instance 0 (8 samples), L=4")
    scn = generate(fam(30, 2.0), 64, 2, seed=4000, horizon=b100)
    xi, lam = naive(scn, B100, 1, seed=4000)
    run("c4_inst0_L2", scn, B100, xi, lam, "projection", SolverConfig(max_iters=2, **FIXED),
        note="BASELINE configs[3] instance 0, L=2")

    # The benched configuration itself: C3 instance 0 (8 samples) over the full L=500 of
    # the throughput protocol (~25 min of reference time on one core), the C2 drift-stress
    # case over L=500, C4 over L=100, and two C3 instances at the same L so the GPU test
    # can solve them in ONE launch with an interleaved member->instance map.
    scn = generate(fam(20, 2.0), 32, 2, seed=3000, horizon=b100)
    xi, lam = naive(scn, B100, 8, seed=3000)
    run("c3_inst0_L500", scn, B100, xi, lam, "projection", SolverConfig(max_iters=500, **FIXED),
        note="BASELINE configs[2] instance 0 (8 samples), the benched L=500")
    scn = generate(fam(10, 1.0), 16, 2, seed=2001, horizon=b100)
    xi, lam = naive(scn, B100, 4, seed=2001)
    run("c2_inst0_L500", scn, B100, xi, lam, "projection", SolverConfig(max_iters=500, **FIXED),
        note="16/10 in [-1,1], L=500: the FP-drift stress case at the full iteration count")
    scn = generate(fam(30, 2.0), 64, 2, seed=4000, horizon=b100)
    xi, lam = naive(scn, B100, 1, seed=4000)
    run("c4_inst0_L100", scn, B100, xi, lam, "projection", SolverConfig(max_iters=100, **FIXED),
        note="BASELINE configs[3] instance 0, L=100")
    for i in (0, 1):
        scn = generate(fam(20, 2.0), 32, 2, seed=3100 + i, horizon=b100)
        xi, lam = naive(scn, B100, 4, seed=3100 + i, lam_scale=0.3, lam_seed=3100 + i)
        run(f"c3pair_inst{i}_L40", scn, B100, xi, lam, "projection",
            SolverConfig(max_iters=40, **FIXED),
            note="one of two C3 instances solved together in one launch by the GPU test")
    # a batch whose members stop on different predicates: member 1 on the fixed-point
    # residual (converged_fp, solver.py:320-322), the others on the primal residual
    scn = generate(fam(3, 1.5), 8, 2, seed=11, horizon=B50.config)
    xi, lam = naive(scn, B50, 3, seed=11)
    run("fp_converge_obs8", scn, B50, xi, lam, "projection",
        SolverConfig(max_iters=20000, primal_tol=1e-9, fp_tol=1e-8),
        note="member 1 ends converged_fp at iteration 290")

    # obstacles, smoothness, rho, rest_to_rest, 3D, moving obstacles
    scn = generate(fam(3, 1.5), 8, 2, seed=11, horizon=B50.config)
    xi, lam = naive(scn, B50, 3, seed=11, lam_scale=0.3)
    run("obs8_projection", scn, B50, xi, lam, "projection", SolverConfig(max_iters=100, **FIXED))
    run("obs8_smoothness", scn, B50, xi, lam, "smoothness", SolverConfig(max_iters=100, **FIXED))
    run("obs8_rho2p5", scn, B50, xi, lam, "projection",
        SolverConfig(rho=2.5, max_iters=100, **FIXED))
    run("obs8_free_ends", scn, B50, xi, lam, "projection", SolverConfig(max_iters=100, **FIXED),
        rest_to_rest=False)
    scn3 = generate(fam(2, 1.5), 6, 3, seed=12, horizon=B50.config)
    xi, lam = naive(scn3, B50, 2, seed=12, lam_scale=0.3)
    run("d3_projection", scn3, B50, xi, lam, "projection", SolverConfig(max_iters=100, **FIXED))
    run("d3_smoothness", scn3, B50, xi, lam, "smoothness", SolverConfig(max_iters=100, **FIXED))
    # 3D spheroid robots (a != b) and moving obstacles
    base = generate(fam(0, 1.5), 4, 3, seed=13, horizon=B50.config)
    scn3b = Scenario(n=4, n_d=3, radii=[0.12, 0.12, 0.06], starts=base.starts, goals=base.goals,
                     obstacles=[Obstacle(center=[0.0, 0.0, 0.0], radii=[0.3, 0.3, 0.2],
                                         velocity=[0.05, -0.04, 0.01])],
                     p_min=base.p_min, p_max=base.p_max, horizon=B50.config)
    xi, lam = naive(scn3b, B50, 2, seed=13, lam_scale=0.3)
    run("d3_spheroid_moving", scn3b, B50, xi, lam, "projection",
        SolverConfig(max_iters=100, **FIXED))
    base = generate(fam(0, 1.5), 6, 2, seed=14, horizon=B50.config)
    scn_m = Scenario(n=6, n_d=2, radii=[0.1] * 3, starts=base.starts, goals=base.goals,
                     obstacles=[Obstacle(center=[-0.4, 0.3], radii=[0.25] * 3, velocity=[0.1, -0.05]),
                                Obstacle(center=[0.5, -0.2], radii=[0.2] * 3, velocity=[-0.08, 0.0])],
                     p_min=base.p_min, p_max=base.p_max, horizon=B50.config)
    xi, lam = naive(scn_m, B50, 3, seed=14, lam_scale=0.3)
    run("moving_obstacles", scn_m, B50, xi, lam, "projection", SolverConfig(max_iters=100, **FIXED))

    # convergence-mode cases of the reference tests (test_solver.py:81-92, 182-217)
    for seed in (1, 2, 3):
        scn = swap(seed)
        st = cold_start(scn, assemble(scn, B50))
        run(f"swap{seed}_converge", scn, B50, st.xi, st.lam, "projection",
            SolverConfig(max_iters=5000))
    scn = swap(3)
    rng = np.random.default_rng(1)
    base = straight_line_coeffs(scn.starts, scn.goals, 11)
    cands = []
    for _ in range(4):
        noise = np.zeros_like(base)
        noise[:, :, 1:-1] = 0.2 * rng.standard_normal(noise[:, :, 1:-1].shape)
        cands.append(base + noise)
    xi = stack_xi(cands)
    run("swap3_batch4_converge", scn, B50, xi, np.zeros_like(xi), "projection",
        SolverConfig(max_iters=2000))
    # smoothness convergence on a mildly interacting instance (test_solver.py:139-146)
    scn = generate(ScenarioFamily(kind="random_box"), n=2, n_d=2, seed=1)
    st = cold_start(scn, assemble(scn, B50))
    run("smooth_nlp_converge", scn, B50, st.xi, st.lam, "smoothness", SolverConfig(max_iters=15000))

    # known answers: overlap (test_solver.py:246-259), workspace (:262-274), coincident
    a = DEFAULT_MARGIN * 0.2
    scn = Scenario(n=2, n_d=2, radii=[0.1] * 3, starts=[[0.0, 0.0], [0.9 * a, 0.0]],
                   goals=[[0.0, 0.0], [0.9 * a, 0.0]], obstacles=[], p_min=[-1, -1], p_max=[1, 1])
    c = straight_line_coeffs(scn.starts, scn.goals, 11)
    st = state_from_xi(xi_from_coeffs(c))
    run("known_overlap", scn, B50, st.xi, st.lam, "projection", SolverConfig(max_iters=3, **FIXED),
        note="primal[0] = 0.1*a*sqrt(K+1)")
    scn = Scenario(n=1, n_d=2, radii=[0.1] * 3, starts=[[0.0, 0.0]], goals=[[0.5, 0.0]],
                   obstacles=[], p_min=[-1, -1], p_max=[1, 1])
    c = straight_line_coeffs(scn.starts + [1.5, 0.0], scn.goals + [1.5, 0.0], 11)
    st = state_from_xi(xi_from_coeffs(c))
    run("known_workspace", scn, B50, st.xi, st.lam, "projection", SolverConfig(max_iters=3, **FIXED))
    scn = Scenario(n=3, n_d=2, radii=[0.1] * 3, starts=[[-0.5, 0.0], [-0.5, 0.0], [0.0, 0.6]],
                   goals=[[0.5, 0.0], [0.5, 0.0], [0.0, -0.6]], obstacles=[],
                   p_min=[-1, -1], p_max=[1, 1])
    c = straight_line_coeffs(scn.starts, scn.goals, 11)
    st = state_from_xi(xi_from_coeffs(c))
    run("known_coincident", scn, B50, st.xi, st.lam, "projection", SolverConfig(max_iters=20, **FIXED),
        note="robots 0 and 1 coincide exactly at every step of the input (alpha=0 rule)")

    # S1-style single steps from random states (trainer/tests/test_acceptance.py:35-87)
    for label, scn in (("2d", generate(ScenarioFamily("random_box"), n=3, n_d=2, seed=1)),
                       ("2d_obstacles", generate(ScenarioFamily("random_box", n_obstacles=2),
                                                 n=2, n_d=2, seed=2)),
                       ("3d", generate(ScenarioFamily("random_box"), n=2, n_d=3, seed=3))):
        if not want(f"step_{label}"):
            continue
        sys_ = assemble(scn, B50)
        d = sys_.dims
        rng = np.random.default_rng(5)
        xi = 0.5 * rng.standard_normal((d.n_d, d.nvar_ax, 8))
        lam = 0.5 * rng.standard_normal((d.n_d, d.nvar_ax, 8))
        tgt = 0.3 * rng.standard_normal(xi.shape)
        mode = ObjectiveMode.projection(tgt)
        cfg = SolverConfig(max_iters=1, **FIXED)
        st = SolverState(xi=xi, lam=lam)
        res = solve_batch(st, sys_, mode, cfg)
        nxt = fixed_point_step(st, sys_, mode, cfg)
        assert np.allclose(np.stack([r.xi for r in res], -1), nxt.xi, rtol=0, atol=1e-12)
        save(f"step_{label}", sys_, mode, st, cfg, res, note="single fixed_point_step")


if __name__ == "__main__":
    main()
