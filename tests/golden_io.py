"""Load a golden fixture (tests/golden/*.npz, written by make_golden.py from the
reference) back into solver inputs. Used by the CPU oracle tests and the GPU
parity tests; nothing here reads /root/reference."""

from __future__ import annotations

import glob
import os
from dataclasses import dataclass

import numpy as np

from paper_2510_09204_b200.problem import (
    BasisConfig, BasisMatrices, ConstraintSystem, SystemDims,
)

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATUS_NAMES = {0: "max_iters", 1: "converged_primal", 2: "converged_fp"}


@dataclass
class Golden:
    name: str
    sys: ConstraintSystem
    kind: str
    target: np.ndarray | None     # (n_d, nv, B) or None
    xi0: np.ndarray               # (n_d, nv, B)
    lam0: np.ndarray
    rho: float
    max_iters: int
    primal_tol: float
    fp_tol: float
    d_max: float
    out: dict                     # reference outputs
    note: str


def names():
    """Solver fixtures (metrics_*.npz / plan_*.npz / stepvars_*.npz belong to the epilogue,
    planner and fixed_point_step-analysis tests)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith(("metrics_", "plan_", "stepvars_")))


def load(name: str) -> Golden:
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    n, n_d, n_basis, K1, n_obs, a_rows, g_rows = (int(v) for v in z["dims"])
    cfg = BasisConfig(n_basis, K1, float(z["duration"]))
    basis = BasisMatrices(W=z["W"], Wd=z["Wd"], Wdd=z["Wdd"], grid=z["grid"], config=cfg)
    n_pairs = n * (n - 1) // 2
    dims = SystemDims(n=n, n_d=n_d, n_basis=n_basis, num_steps=K1, n_obs=n_obs,
                      n_pairs=n_pairs, rows_pairs=n_pairs * K1, rows_obs=n * n_obs * K1,
                      nvar_ax=n * n_basis, a_rows=a_rows, g_rows=g_rows)
    sys_ = ConstraintSystem(A=z["A"], b=z["b"], h=z["h"], pair_axes=z["pair_axes"],
                            obs_axes=z["obs_axes"], obs_pos=z["obs_pos"], dims=dims,
                            basis=basis, d_max=float(z["d_max"]))
    rho, max_iters, ptol, ftol, d_max = z["cfg"]
    kind = str(z["kind"])
    T = z["out_trace"]
    its = z["out_iterations"]
    out = {
        "xi": z["out_xi"], "lam": z["out_lam"],
        "status": [STATUS_NAMES[int(s)] for s in z["out_status"]],
        "iterations": its, "primal": z["out_primal"], "eq_max": z["out_eq"],
        "trace": [T[b, : its[b] + 1] for b in range(T.shape[0])],
    }
    return Golden(name=name, sys=sys_, kind=kind,
                  target=z["target"] if kind == "projection" else None,
                  xi0=z["xi0"], lam0=z["lam0"], rho=float(rho), max_iters=int(max_iters),
                  primal_tol=float(ptol), fp_tol=float(ftol), d_max=float(d_max), out=out,
                  note=str(z["note"]))


def manifest() -> dict:
    import json
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as fh:
        return json.load(fh)


def assert_properties(out: dict, g: "Golden"):
    """Property parity for round-off-determined (chaotic) cases: same status,
    residual below tolerance when converged, exact boundary equalities and an
    iteration count within a band of the reference's (test_solver.py:81-92,
    288-293; test_acceptance.py P4)."""
    for b in range(len(g.out["iterations"])):
        assert out["status"][b] == g.out["status"][b], (b, out["status"][b], g.out["status"][b])
        if g.out["status"][b] == "converged_primal":
            assert float(out["primal"][b]) < g.primal_tol
        assert float(out["eq_max"][b]) < 1e-8
        ref_its = int(g.out["iterations"][b])
        assert abs(int(out["iterations"][b]) - ref_its) <= 0.3 * ref_its + 10, \
            (b, out["iterations"][b], ref_its)


def compare(got: dict, ref: dict):
    """Worst-case errors between two solve outputs (member-major dicts).

    xi_rel: per member max|dxi| / max|xi_ref|; lam_abs; primal/trace abs.
    fp_abs / fp_rel: the fixed-point column trace[:, 1] (solver.py:316, 329-333):
    absolute error and error relative to max(|fp_ref|, 1e-12) over the finite
    entries; the first entry (+inf, before any step) must be +inf on both sides.
    In fixed-iteration mode iterations and status must match exactly."""
    B = len(ref["iterations"])
    flat = lambda v: np.asarray(v).reshape(-1)
    xi_rel = lam_abs = trace_abs = final_abs = eq_abs = fp_abs = fp_rel = 0.0
    same_its = True
    fp_inf_ok = True
    for b in range(B):
        xr = flat(ref["xi"][b])
        xi_rel = max(xi_rel, float(np.abs(flat(got["xi"][b]) - xr).max()
                                   / max(np.abs(xr).max(), 1e-300)))
        lam_abs = max(lam_abs, float(np.abs(flat(got["lam"][b]) - flat(ref["lam"][b])).max()))
        tg, tr = np.asarray(got["trace"][b]), np.asarray(ref["trace"][b])
        L = min(len(tg), len(tr))
        trace_abs = max(trace_abs, float(np.abs(tg[:L, 0] - tr[:L, 0]).max()))
        if L:
            fp_inf_ok &= bool(np.isposinf(tg[0, 1]) and np.isposinf(tr[0, 1]))
        if L > 1:
            fg, fr = tg[1:L, 1], tr[1:L, 1]
            fp_inf_ok &= bool(np.all(np.isfinite(fg)) and np.all(np.isfinite(fr)))
            dfp = np.abs(fg - fr)
            fp_abs = max(fp_abs, float(dfp.max()))
            fp_rel = max(fp_rel, float((dfp / np.maximum(np.abs(fr), 1e-12)).max()))
        final_abs = max(final_abs, abs(float(got["primal"][b]) - float(ref["primal"][b])))
        eq_abs = max(eq_abs, abs(float(got["eq_max"][b]) - float(ref["eq_max"][b])))
        same_its &= int(got["iterations"][b]) == int(ref["iterations"][b]) and \
            got["status"][b] == ref["status"][b]
    return dict(xi_rel=xi_rel, lam_abs=lam_abs, trace_abs=trace_abs, final_abs=final_abs,
                eq_abs=eq_abs, same_iterations=same_its, fp_abs=fp_abs, fp_rel=fp_rel,
                fp_inf_ok=fp_inf_ok)
