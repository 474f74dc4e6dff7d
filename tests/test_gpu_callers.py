"""GPU tests of the callers either side of the SF: stage-1 residual
ranking (pipeline.py:113-115), on-device handoff from PyTorch producers, and the
time-scaling epilogue (basis.py:119-142)."""

import numpy as np
import pytest

import golden_io
from oracle import sf_kron

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_09204_b200 import solver  # noqa: E402
from paper_2510_09204_b200.problem import (  # noqa: E402
    BasisConfig, ScenarioFamily, assemble, build_basis, generate, sample_naive_prior, stack_xi,
)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["c2_infeasible_L60", "c3_inst0_L4", "d3_spheroid_moving",
                                  "moving_obstacles", "known_overlap", "known_workspace"])
def test_batch_primal_residual_matches_reference_trace0(name):
    """trace[0, 0] of the reference solve is the primal residual of the warm start."""
    g = golden_io.load(name)
    pre = solver.batch_primal_residual(g.xi0, g.sys)
    ref = np.array([t[0, 0] for t in g.out["trace"]])
    assert np.abs(pre - ref).max() < 1e-9


def test_rank_candidates_matches_oracle_order():
    basis = build_basis(BasisConfig(11, 50, 5.0))
    scn = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=3), 8, 2, seed=5,
                   horizon=basis.config)
    sys_ = assemble(scn, basis)
    xi = stack_xi(sample_naive_prior(scn, basis, 64, seed=5))
    pre, order = solver.rank_candidates(xi, sys_)
    sf = sf_kron.KronSF(sys_, "projection", 1.0)
    _, ref, _ = sf.analyze(sf_kron.to_member_major(xi, 8, 11))
    assert np.abs(pre - ref).max() < 1e-10
    assert np.array_equal(order, np.argsort(ref, kind="stable"))


def test_device_tensor_handoff_matches_host_path():
    """CUDA tensors from a PyTorch producer go straight into the solve (no host copy)."""
    g = golden_io.load("obs8_projection")
    d = g.sys.dims
    mm = solver.to_member_major(g.xi0, d.n, d.n_basis)
    lm = solver.to_member_major(g.lam0, d.n, d.n_basis)
    cfg = solver.SolverConfig(max_iters=40)
    host = solver.solve_instances([g.sys], mm, lm, mm, cfg=cfg, fixed_iterations=True)
    dev = torch.device("cuda")
    t_xi = torch.from_numpy(mm).to(dev)
    t_lm = torch.from_numpy(lm).to(dev)
    batch = solver.DeviceBatch([g.sys], t_xi, t_lm, t_xi, cfg=cfg, early_exit=False)
    assert batch.h2d_bytes < mm.nbytes          # only the instance data crossed PCIe
    batch.launch()
    out = batch.results()
    assert np.array_equal(out["xi"], host.xi)


def test_time_scale_matches_numpy_reference():
    basis = build_basis(BasisConfig(11, 50, 5.0))
    scn = generate(ScenarioFamily("random_box"), 6, 2, seed=3, horizon=basis.config)
    cands = sample_naive_prior(scn, basis, 5, seed=3)
    dense = build_basis(BasisConfig(11, 10 * 49 + 1, 5.0))
    mm = np.stack([c.transpose(1, 0, 2) for c in cands])
    vhat, ahat = solver.kinematic_peaks(mm, basis)
    for b, c in enumerate(cands):
        v = np.linalg.norm(np.einsum("kc,ndc->nkd", dense.Wd, c), axis=2).max()
        a = np.linalg.norm(np.einsum("kc,ndc->nkd", dense.Wdd, c), axis=2).max()
        assert abs(vhat[b] - v) < 1e-12 * max(1.0, v) and abs(ahat[b] - a) < 1e-12 * max(1.0, a)
    gamma, scaled = solver.time_scale_for_limits(cands[1], basis, v_max=0.3, a_max=0.5)
    v = np.linalg.norm(np.einsum("kc,ndc->nkd", dense.Wd, cands[1]), axis=2).max()
    a = np.linalg.norm(np.einsum("kc,ndc->nkd", dense.Wdd, cands[1]), axis=2).max()
    assert abs(gamma - max(1.0, v / 0.3, np.sqrt(a / 0.5))) < 1e-12 * gamma
    assert abs(scaled.config.duration - gamma * 5.0) < 1e-12
