"""Pin the CPU oracle (oracle/sf_dense.py, oracle/sf_kron.py) to the reference's
own outputs stored in tests/golden/*.npz. CPU only.

Cases marked 'chaotic' in tests/golden/manifest.json (symmetric cold-start
swaps whose symmetry breaks on round-off; see classify.py) are checked through
the reference tests' properties instead of trajectory equality."""

import numpy as np
import pytest

import golden_io
from oracle import sf_dense, sf_kron

# the dense restatement is slow at the C3/C4 shapes: those go through the
# Kronecker restatement only in the default suite
DENSE_SKIP = {"c3_inst0_L4", "c4_inst0_L2", "c3_inst0_L500", "c2_inst0_L500", "c4_inst0_L100",
              "c3pair_inst0_L40", "c3pair_inst1_L40"}
# the Kronecker restatement needs minutes for these (C3 x 8 samples x 501 evaluations):
# the CPU suite checks a truncated prefix of their trace; the full run is the GPU parity test
KRON_PREFIX = {"c3_inst0_L500": 40, "c2_inst0_L500": 120, "c4_inst0_L100": 12}
MANIFEST = golden_io.manifest()


def _run(mod, g, **kw):
    return mod.solve_batch(g.sys, g.xi0, g.lam0, kind=g.kind, target=g.target, rho=g.rho,
                           max_iters=g.max_iters, primal_tol=g.primal_tol, fp_tol=g.fp_tol, **kw)


def _check(name, out, g, xi_tol):
    info = MANIFEST[name]
    if info["class"] == "chaotic":
        golden_io.assert_properties(out, g)
        return
    err = golden_io.compare(out, g.out)
    assert err["same_iterations"], err
    assert err["xi_rel"] < xi_tol, err
    if info["class"] != "lam_degenerate":
        assert err["lam_abs"] < 1e-7, err
        # fixed-point column trace[:, 1] (its ||dlambda||^2 term is what lam_degenerate lacks)
        assert err["fp_inf_ok"] and err["fp_rel"] < 1e-6, err
    assert err["trace_abs"] < 1e-9, err
    assert err["eq_abs"] < 1e-9, err


@pytest.mark.parametrize("name", golden_io.names())
def test_kron_oracle_matches_reference(name):
    g = golden_io.load(name)
    if name in KRON_PREFIX:
        L = KRON_PREFIX[name]
        out = sf_kron.solve_batch(g.sys, g.xi0, g.lam0, kind=g.kind, target=g.target, rho=g.rho,
                                  max_iters=L, primal_tol=g.primal_tol, fp_tol=g.fp_tol,
                                  early_exit=False)
        for b in range(len(out["trace"])):
            tg, tr = out["trace"][b], g.out["trace"][b][: L + 1]
            assert np.abs(tg[:, 0] - tr[:, 0]).max() < 1e-9
            assert np.all(np.abs(tg[1:, 1] - tr[1:, 1]) < 1e-6 * np.maximum(np.abs(tr[1:, 1]), 1e-12))
        return
    out = _run(sf_kron, g, early_exit=not MANIFEST[name]["fixed_iterations"])
    # the reference itself drifts ~1e-9 over 500 noise-level iterations (c1)
    _check(name, out, g, 1e-7)


@pytest.mark.parametrize("name", [n for n in golden_io.names() if n not in DENSE_SKIP])
def test_dense_oracle_matches_reference(name):
    g = golden_io.load(name)
    _check(name, _run(sf_dense, g), g, 1e-9)


def test_known_answer_overlap_primal():
    """test_solver.py:246-259: overlapping pair -> primal = 0.1 a sqrt(K+1)."""
    g = golden_io.load("known_overlap")
    a = 1.1 * 0.2
    expect = 0.1 * a * np.sqrt(g.sys.dims.num_steps)
    assert abs(g.out["trace"][0][0, 0] - expect) < 1e-9
    out = _run(sf_kron, g, early_exit=False)
    assert abs(out["trace"][0][0, 0] - expect) < 1e-9


def test_kkt_blocks_match_dense_inverse():
    import scipy.linalg
    for name, kind in (("obs8_projection", "projection"), ("d3_smoothness", "smoothness"),
                       ("obs8_free_ends", "projection")):
        g = golden_io.load(name)
        d = g.sys.dims
        sf = sf_kron.KronSF(g.sys, kind, 1.0)
        F, G, _ = sf_dense.dense_operators(d.n, d.n_obs, g.sys.basis.W)
        kkt = sf_dense.DenseKkt(F, G, g.sys.A, g.sys.basis.Wdd, d.n, kind, 1.0)
        Minv = scipy.linalg.lu_solve(kkt.lu, np.eye(kkt.size))
        nv, n = d.nvar_ax, d.n
        Mxx = np.kron(np.eye(n), sf.Pxx) + np.kron(np.ones((n, n)) / n, sf.Rxx - sf.Pxx)
        Mxb = np.kron(np.eye(n), sf.Pxb) + np.kron(np.ones((n, n)) / n, sf.Rxb - sf.Pxb)
        scale = np.abs(Minv).max()
        assert np.abs(Minv[:nv, :nv] - Mxx).max() < 1e-12 * scale
        assert np.abs(Minv[:nv, nv:] - Mxb).max() < 1e-12 * scale
        M = np.linalg.inv(Minv)
        assert abs(np.linalg.cond(M) / sf.cond - 1) < 1e-6


# ------------------------------------------------------------------ metrics epilogue (§8 f4)
def _metrics_cases():
    import glob
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(here, "metrics_*.npz")))


def load_metrics_golden(name):
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz"))
    nd = int(z["n_d"])
    obs = [(o[0, :nd], o[1, :nd], o[2, :nd]) for o in z["obstacles"]]
    return z, nd, obs


def metrics_close(got, ref, rtol=1e-12):
    got, ref = np.asarray(got), np.asarray(ref)
    assert np.array_equal(np.isinf(got), np.isinf(ref))
    fin = np.isfinite(ref)
    err = np.abs(got[fin] - ref[fin])
    assert (err <= rtol * np.maximum(1.0, np.abs(ref[fin]))).all(), (got, ref)


@pytest.mark.parametrize("name", _metrics_cases())
def test_metrics_oracle_matches_reference(name):
    """oracle/metrics.py against compute_metrics outputs of the reference (metrics.py:48-87)."""
    from oracle.metrics import trajectory_metrics
    z, nd, obs = load_metrics_golden(name)
    assert len(_metrics_cases()) >= 5
    for c, m in zip(z["coeffs"], z["metrics"]):
        got = trajectory_metrics(c, int(z["n_basis"]), int(z["num_steps"]), float(z["duration"]),
                                 obs, int(z["dense_factor"]))
        metrics_close(got, m)


def test_kron_oracle_matches_live_reference_on_random_problems():
    """Where the reference package is importable (this build container), a few random small
    problems through its own generator / assemble / solve_batch against oracle/sf_kron.py
    (oracle/fuzz_vs_reference.py runs the longer campaign)."""
    import os
    import subprocess
    import sys
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference package not present")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=ref_src, PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, os.path.join(root, "oracle", "fuzz_vs_reference.py"), "6", "11"],
                         capture_output=True, text=True, env=env, cwd="/tmp", timeout=600)
    if "No module named" in out.stderr:
        pytest.skip("reference dependencies missing")
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]


# ------------------------------------------------------------------ fixed_point_step vars / s (§8 a15)
def load_stepvars(name):
    import os
    z = np.load(os.path.join(golden_io.GOLDEN_DIR, f"stepvars_{name}.npz"), allow_pickle=False)
    from paper_2510_09204_b200.problem import BasisConfig, BasisMatrices, ConstraintSystem, SystemDims
    n, n_d, n_basis, K1, n_obs, a_rows, g_rows = (int(v) for v in z["dims"])
    basis = BasisMatrices(W=z["W"], Wd=z["Wd"], Wdd=z["Wdd"], grid=z["grid"],
                          config=BasisConfig(n_basis, K1, float(z["duration"])))
    P = n * (n - 1) // 2
    dims = SystemDims(n=n, n_d=n_d, n_basis=n_basis, num_steps=K1, n_obs=n_obs, n_pairs=P,
                      rows_pairs=P * K1, rows_obs=n * n_obs * K1, nvar_ax=n * n_basis,
                      a_rows=a_rows, g_rows=g_rows)
    sys_ = ConstraintSystem(A=z["A"], b=z["b"], h=z["h"], pair_axes=z["pair_axes"],
                            obs_axes=z["obs_axes"], obs_pos=z["obs_pos"], dims=dims, basis=basis,
                            d_max=float(z["d_max"]))
    return z, sys_


STEPVARS = ("2d_obstacles", "3d", "obs8")


@pytest.mark.parametrize("name", STEPVARS)
def test_dense_oracle_step_vars_match_reference(name):
    """oracle/sf_dense.py's spherical variables and slack of a step's input iterate against
    the reference's fixed_point_step(...).vars / .s (tests/golden/make_stepvars_golden.py)."""
    z, sys_ = load_stepvars(name)
    sf = sf_dense.DenseSF(sys_, "projection", 1.0)
    (al, be, dd), (alo, beo, do), s = sf.spherical_vars(z["xi0"])
    for got, key in ((al, "alpha"), (be, "beta"), (dd, "d"), (alo, "alpha_o"), (beo, "beta_o"),
                     (do, "d_o"), (s, "out_s")):
        assert got.shape == z[key].shape, key
        assert np.abs(got - z[key]).max() <= 1e-12 * max(1.0, np.abs(z[key]).max()), key
