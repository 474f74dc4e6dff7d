"""Randomized parity campaign: random shapes / modes / parameters, GPU solve vs the FP64
Kronecker oracle (oracle/sf_kron.py). Test infrastructure (imports the oracle).
    python tools/fuzz_parity.py [cases] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import sf_kron  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble,  # noqa: E402
                                           build_basis, generate, sample_naive_prior, stack_xi)


def one(rng, case):
    import dataclasses
    big = rng.random() < BIG_FRAC
    n = int(rng.choice([48, 64, 80, 128])) if big else int(rng.choice([1, 2, 3, 5, 8, 12, 16, 20, 31, 32, 33, 40]))
    n_d = int(rng.choice([2, 2, 2, 3]))
    nxi = int(rng.integers(6, 13))
    K1 = int(rng.integers(max(nxi, 12), 110))
    m = int(rng.choice([0, 0, 1, 3, 7, 15, 31]))
    kind = "projection" if rng.random() < 0.8 else "smoothness"
    rho = float(rng.choice([0.5, 1.0, 2.5]))
    d_max = float(rng.choice([1e6, 1e6, 50.0, 4.0]))
    S = int(rng.integers(1, 5))
    h = max(1.0, 2.0 * (n / 32) ** 0.5) * float(rng.choice([1.0, 1.5]))
    basis = build_basis(BasisConfig(nxi, K1, 5.0))
    fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-h, h), n_obstacles=m)
    try:
        scn = generate(fam, n, n_d, seed=int(rng.integers(1 << 30)), horizon=basis.config)
    except Exception as e:   # generator cannot place this configuration
        return None, f"skip ({type(e).__name__})"
    sys_ = dataclasses.replace(assemble(scn, basis), d_max=d_max)
    moving = m > 0 and rng.random() < MOVING_FRAC
    if moving:   # linear obstacle tracks c + v t_k (per-step obstacle rows, no grid)
        op = np.array(sys_.obs_pos, float)
        v = 0.3 * rng.standard_normal(op.shape[:2])
        t = np.linspace(0.0, 1.0, op.shape[2])
        sys_ = dataclasses.replace(sys_, obs_pos=op[:, :, :1] + v[:, :, None] * t[None, None, :])
    xi = stack_xi(sample_naive_prior(scn, basis, S, seed=case))
    lam = 0.3 * np.random.default_rng(case).standard_normal(xi.shape)
    mm = lambda x: solver.to_member_major(x, n, nxi)
    L = int(rng.integers(1, 12 if big else 60))
    fixed = rng.random() < 0.7
    cfg = solver.SolverConfig(rho=rho, max_iters=L, primal_tol=1e-3 if not fixed else 1e-3)
    cluster = int(rng.choice([0, 1, 2, 4]))
    from paper_2510_09204_b200.errors import ShapeError
    try:
        got = solver.solve_instances([sys_], mm(xi), mm(lam), mm(xi) if kind == "projection" else None,
                                     kind=kind, cfg=cfg, fixed_iterations=fixed, cluster=cluster)
    except ShapeError as e:   # an explicit cluster size this layout cannot hold (auto falls back)
        if cluster > 0 and "cluster" in str(e):
            return None, f"skip (n={n} m={m} cluster={cluster}: {e})"
        if "exceed shared memory" in str(e):   # documented limit (moving obstacles at large n)
            return None, f"skip (n={n} n_d={n_d} m={m}: {e})"
        raise
    ref = sf_kron.solve_batch(sys_, xi, lam, kind=kind, target=xi if kind == "projection" else None,
                              rho=rho, max_iters=L, early_exit=not fixed)
    worst = 0.0
    for b in range(S):
        r = np.asarray(ref["xi"][b]).reshape(-1)
        rel = np.abs(got.xi[b].reshape(-1) - r).max() / max(np.abs(r).max(), 1e-300)
        if not fixed and int(got.iterations[b]) != int(ref["iterations"][b]):
            return False, f"iterations {got.iterations[b]} vs {ref['iterations'][b]}"
        tr = np.abs(got.trace[b][:, 0] - ref["trace"][b][:, 0]).max()
        worst = max(worst, rel, tr)
    desc = (f"n={n} n_d={n_d} nxi={nxi} K1={K1} m={m}{' moving' if moving else ''} {kind} rho={rho} "
            f"d_max={d_max:g} S={S} L={L} "
            f"{'fixed' if fixed else 'converge'} cluster={cluster}")
    return worst < 1e-8, f"{desc}: worst {worst:.2e}"


BIG_FRAC, MOVING_FRAC = 0.0, 0.0


def main():
    global BIG_FRAC, MOVING_FRAC
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    BIG_FRAC = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0       # share of n in 48..128
    MOVING_FRAC = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0    # share with moving obstacles
    rng = np.random.default_rng(seed)
    bad = 0
    for c in range(cases):
        ok, msg = one(rng, c)
        if ok is None:
            print("   ", msg)
            continue
        print("ok " if ok else "BAD", msg, flush=True)
        bad += 0 if ok else 1
    print(f"{bad} bad of {cases}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
