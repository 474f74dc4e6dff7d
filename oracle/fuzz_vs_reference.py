"""ORACLE PINNING (test infrastructure; runs only where /root/reference is importable):
random small problems through the reference's own generator, assemble and solve_batch
(swarmplan, pkg/src/swarmplan/solver.py:286-355) against oracle/sf_kron.py.
    PYTHONPATH=/root/reference/pkg/src python oracle/fuzz_vs_reference.py [cases] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from oracle import sf_kron  # noqa: E402


def main():
    from swarmplan.basis import BasisConfig, build_basis
    from swarmplan.constraints import assemble
    from swarmplan.errors import GenerationError
    from swarmplan.pipeline import sample_naive_prior
    from swarmplan.scenario import ScenarioFamily, generate
    from swarmplan.solver import ObjectiveMode, SolverConfig, SolverState, solve_batch, stack_xi

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    bad = done = 0
    for c in range(cases):
        n = int(rng.choice([1, 2, 3, 4, 6]))
        n_d = int(rng.choice([2, 2, 3]))
        nxi = int(rng.integers(6, 12))
        K1 = int(rng.integers(max(12, nxi), 40))
        m = int(rng.choice([0, 1, 2, 4]))
        kind = "projection" if rng.random() < 0.75 else "smoothness"
        rho = float(rng.choice([0.5, 1.0, 2.0]))
        d_max = float(rng.choice([1e6, 1e6, 3.0]))
        L = int(rng.integers(1, 12))
        basis = build_basis(BasisConfig(nxi, K1, 5.0))
        fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-1.0, 1.0), n_obstacles=m)
        try:
            scn = generate(fam, n, n_d, seed=int(rng.integers(1 << 30)), horizon=basis.config)
        except GenerationError:
            continue
        sys_ = assemble(scn, basis, d_max=d_max)
        cand = sample_naive_prior(scn, basis, 2, seed=c)
        xi = stack_xi(cand.candidates)
        lam = 0.3 * np.random.default_rng(c).standard_normal(xi.shape)
        mode = ObjectiveMode.projection(xi) if kind == "projection" else ObjectiveMode.smoothness()
        cfg = SolverConfig(rho=rho, max_iters=L, primal_tol=1e-300, fp_tol=1e-300)
        ref = solve_batch(SolverState(xi=xi.copy(), lam=lam.copy()), sys_, mode, cfg)
        orc = sf_kron.solve_batch(sys_, xi, lam, kind=kind, target=xi if kind == "projection" else None,
                                  rho=rho, max_iters=L, early_exit=False)
        worst = 0.0
        for b, r in enumerate(ref):
            o = orc
            if r.iterations != L:
                # the reference stops on an exactly-zero residual even at tol 1e-300:
                # compare with the oracle run to the same iteration
                o = sf_kron.solve_batch(sys_, xi[:, :, b:b + 1], lam[:, :, b:b + 1], kind=kind,
                                        target=xi[:, :, b:b + 1] if kind == "projection" else None,
                                        rho=rho, max_iters=r.iterations, early_exit=False)
                bo = 0
            else:
                bo = b
            x = np.asarray(o["xi"][bo]).reshape(-1)
            rx = np.asarray(r.xi).reshape(-1)
            worst = max(worst, np.abs(x - rx).max() / max(np.abs(rx).max(), 1e-300),
                        np.abs(o["trace"][bo][:, 0] - np.asarray(r.trace)[:, 0]).max())
        ok = worst < 1e-10
        bad += 0 if ok else 1
        done += 1
        print(("ok " if ok else "BAD"), f"n={n} n_d={n_d} nxi={nxi} K1={K1} m={m} {kind} rho={rho} "
              f"d_max={d_max:g} L={L}: worst {worst:.2e}", flush=True)
    print(f"{bad} bad of {done}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
