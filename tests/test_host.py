"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/sfb.h declares, input validation mirrors the reference's errors, the
problem model reproduces the reference generator, and the layout helpers."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest

import golden_io
from paper_2510_09204_b200 import _lib, solver
from paper_2510_09204_b200.errors import SetupError, ShapeError, UsageError
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble, build_basis,
                                           generate, sample_naive_prior, stack_xi)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sfb.h")).read()
    decl = set(re.findall(r"^\s*(?:const\s+)?[\w ]+?\**\s*\b(sfb_\w+)\s*\(", hdr, re.M))
    assert decl >= {"sfb_plan_create", "sfb_solve", "sfb_plan_destroy", "sfb_last_error"}
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in decl:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) == decl
    assert _lib.lib().sfb_abi_version() == 1


def test_struct_layouts_match_header():
    """ctypes mirrors of sfb_dims / sfb_batch / sfb_config / sfb_out (field order and sizes)."""
    hdr = open(os.path.join(ROOT, "include", "sfb.h")).read()
    for cname, cls in (("sfb_dims", _lib.Dims), ("sfb_batch", _lib.Batch),
                       ("sfb_config", _lib.Config), ("sfb_out", _lib.Out)):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), hdr, re.S).group(1)
        fields = re.findall(r"\b(\w+);", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
        assert fields == [f[0] for f in cls._fields_], (cname, fields)


def test_config_and_mode_validation():
    with pytest.raises(SetupError):
        solver.SolverConfig(rho=0.0)
    with pytest.raises(SetupError):
        solver.SolverConfig(primal_tol=-1.0)
    t = np.zeros((2, 22, 1))
    assert solver._target(solver.ObjectiveMode.projection(t), 4).shape == (2, 22, 4)
    with pytest.raises(ShapeError):
        solver._target(solver.ObjectiveMode.projection(np.zeros((2, 22, 3))), 4)
    assert solver._target(solver.ObjectiveMode.smoothness(), 4) is None


def test_system_data_structure_checks():
    g = golden_io.load("obs8_projection")
    sd = solver.system_data(g.sys)
    assert sd.n_bnd == 6 and sd.E.shape == (6, 11)
    assert np.array_equal(np.kron(np.eye(8), sd.E), g.sys.A)
    assert sd.box.shape == (2, 2)
    import dataclasses
    bad_A = np.vstack([g.sys.A, g.sys.A[:1]])   # test_solver.py:296-307: singular KKT
    bad = dataclasses.replace(g.sys, A=bad_A, b=np.hstack([g.sys.b, g.sys.b[:, :1]]))
    with pytest.raises(SetupError):
        solver.system_data(bad, "smoothness")
    h = g.sys.h.copy()
    h[0, 5] += 0.1
    with pytest.raises(UsageError):
        solver.system_data(dataclasses.replace(g.sys, h=h))


def test_member_major_round_trip():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 5 * 7, 4))
    mm = solver.to_member_major(x, 5, 7)
    assert mm.shape == (4, 3, 5, 7)
    back = np.moveaxis(mm.reshape(4, 3, 35), 0, -1)
    assert np.array_equal(back, x)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_problem_model_reproduces_reference_generator():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    try:
        from swarmplan import basis as rb, constraints as rc, pipeline as rp, scenario as rs
    finally:
        sys.path.remove(REF)
    for (n, m, h, nd, seed) in ((8, 3, 1.5, 2, 11), (32, 20, 2.0, 2, 3000), (6, 2, 1.5, 3, 12)):
        cfg = BasisConfig(11, 100, 5.0)
        ours = generate(ScenarioFamily("random_box", box=(-h, h), n_obstacles=m), n, nd, seed=seed,
                        horizon=cfg)
        ref = rs.generate(rs.ScenarioFamily("random_box", box=(-h, h), n_obstacles=m), n, nd,
                          seed=seed, horizon=rb.BasisConfig(11, 100, 5.0))
        assert np.array_equal(ours.starts, ref.starts) and np.array_equal(ours.goals, ref.goals)
        B1, B2 = build_basis(cfg), rb.build_basis(rb.BasisConfig(11, 100, 5.0))
        for a, b in ((B1.W, B2.W), (B1.Wd, B2.Wd), (B1.Wdd, B2.Wdd)):
            assert np.abs(a - b).max() < 1e-12
        s1 = assemble(ours, B1)
        s2 = rc.assemble(ref, B2)
        assert np.abs(s1.A - s2.A).max() < 1e-12
        assert np.array_equal(s1.b, s2.b) and np.array_equal(s1.h, s2.h)
        assert np.array_equal(s1.obs_pos, s2.obs_pos) and np.array_equal(s1.obs_axes, s2.obs_axes)
        assert np.array_equal(s1.pair_axes, s2.pair_axes)
        c1 = stack_xi(sample_naive_prior(ours, B1, 4, seed=seed))
        c2 = stack_xi(rp.sample_naive_prior(ref, B2, 4, seed=seed).candidates)
        assert np.abs(c1 - c2).max() < 1e-12


def test_bench_roofline_model_numbers():
    import bench
    o32, o64 = bench.algorithmic_ops(32, 20, 100, 11, 2, 6, 0, 1)
    # C3 screened FP32 0.874 M at A = 0, FP64 ~0.184 M
    assert abs(o32 - 873_600) < 1 and abs(o64 - 183_852) < 1


def test_kron_structure_check_matches_dense_kronecker():
    """solver._kron_checked (diagonal blocks + non-zero count) agrees with the dense
    A == kron(I_n, E) comparison it replaced, on exact, perturbed, NaN and misplaced entries."""
    rng = np.random.default_rng(5)
    for n, nb, nx in [(1, 6, 11), (3, 2, 5), (8, 6, 11), (32, 6, 11)]:
        E = rng.standard_normal((nb, nx))
        E[rng.random(E.shape) < 0.3] = 0.0
        A = np.kron(np.eye(n), E)
        assert solver._kron_checked(A, n, E)
        cases = []
        B = A.copy(); B[0, -1] = 1e-300; cases.append(B)                # off-diagonal block
        B = A.copy(); B[-1, 0] = -2.0; cases.append(B)
        B = A.copy(); B[nb - 1, nx - 1] += 1e-12; cases.append(B)       # diagonal block differs
        B = A.copy(); B[0, 0] = np.nan; cases.append(B)
        for B in cases:
            dense = bool(np.array_equal(B, np.kron(np.eye(n), E)))
            assert solver._kron_checked(B, n, E) == dense
        assert not solver._kron_checked(A[:, :-1], n, E)                 # wrong shape


def test_dense_selection_structure_is_checked():
    """a system carrying dense F / G / pair_index (the reference's
    ConstraintSystem) is checked against the structure the Kronecker plan assumes."""
    import dataclasses
    from oracle import sf_dense
    g = golden_io.load("obs8_projection")
    d = g.sys.dims
    F, G, pairs = sf_dense.dense_operators(d.n, d.n_obs, g.sys.basis.W)
    ok = dataclasses.replace(g.sys, F=F, G=G)
    solver._system_data(ok, "projection", 1.0)          # the assemble structure passes
    rows = {0, d.num_steps - 1, d.n_pairs * d.num_steps - 1, d.n_pairs * d.num_steps,
            F.shape[0] - 1, (d.n_pairs // 2) * d.num_steps + d.num_steps // 2}
    F2 = F.copy()
    F2[sorted(rows)[2]] *= 2.0                            # a re-weighted (sampled) pair row
    with pytest.raises(UsageError):
        solver._system_data(dataclasses.replace(g.sys, F=F2, G=G), "projection", 1.0)
    with pytest.raises(UsageError):                      # missing obstacle rows
        solver._system_data(dataclasses.replace(g.sys, F=F[:-d.num_steps], G=G), "projection", 1.0)
    with pytest.raises(UsageError):                      # a box of different sign
        solver._system_data(dataclasses.replace(g.sys, F=F, G=-G), "projection", 1.0)

    import types
    w = types.SimpleNamespace(**{f.name: getattr(g.sys, f.name) for f in dataclasses.fields(g.sys)},
                              pair_index=[(0, 1)])              # a subset of the pairs
    with pytest.raises(UsageError):
        solver._system_data(w, "projection", 1.0)
