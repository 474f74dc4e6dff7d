"""GPU tests of the §8 rows a15 (fixed_point_step returns s and vars) and f3 (producer-layout
handoff), plus the multi-instance member mapping pinned to reference goldens. Marked `gpu`."""

import numpy as np
import pytest

import golden_io
from oracle import sf_kron
from test_oracle import STEPVARS, load_stepvars

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_09204_b200 import solver  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _angle_err(a, b):
    d = np.abs(a - b)
    return np.minimum(d, np.abs(d - 2 * np.pi))   # atan2 at the +-pi cut


@pytest.mark.parametrize("name", STEPVARS)
def test_fixed_point_step_returns_vars_and_slack_of_the_reference(name):
    """solver.py:246-256: SolverState(xi, lam, s=s, vars=vars) — s and vars of the INPUT
    iterate, against the reference's own fixed_point_step outputs."""
    z, sys_ = load_stepvars(name)
    st = solver.SolverState(xi=z["xi0"], lam=z["lam0"])
    nxt = solver.fixed_point_step(st, sys_, solver.ObjectiveMode.projection(z["target"]),
                                  solver.SolverConfig())
    assert np.abs(nxt.xi - z["out_xi"]).max() <= 1e-10 * np.abs(z["out_xi"]).max()
    assert np.abs(nxt.lam - z["out_lam"]).max() <= 1e-10 * max(1.0, np.abs(z["out_lam"]).max())
    assert nxt.s.shape == z["out_s"].shape
    assert np.abs(nxt.s - z["out_s"]).max() <= 1e-12
    v = nxt.vars
    for key in ("alpha", "beta", "alpha_o", "beta_o"):
        got, ref = getattr(v, key), z[key]
        assert got.shape == ref.shape, key
        assert _angle_err(got, ref).max() <= 1e-10, key
    for key in ("d", "d_o"):
        got, ref = getattr(v, key), z[key]
        assert got.shape == ref.shape, key
        assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max(), key


def test_producer_layout_fp32_cuda_handoff():
    """§8 f3: the flow sampler (flow_model.py:228-256) and InitNet.forward (init_net.py:74-96)
    emit (B, n, n_d, n_basis) tensors, FP32 on the GPU. They go in as-is (permuted and widened
    on the device) and solve bitwise like the member-major FP64 copy of the same values."""
    g = golden_io.load("obs8_projection")
    d = g.sys.dims
    B = g.xi0.shape[-1]
    # producer layout (B, n, n_d, n_xi) from the reference layout (n_d, n*n_xi, B)
    prod = np.moveaxis(g.xi0.reshape(d.n_d, d.n, d.n_basis, B), -1, 0).transpose(0, 2, 1, 3)
    lam_p = np.moveaxis(g.lam0.reshape(d.n_d, d.n, d.n_basis, B), -1, 0).transpose(0, 2, 1, 3)
    x32 = torch.from_numpy(np.ascontiguousarray(prod)).float().cuda()
    l32 = torch.from_numpy(np.ascontiguousarray(lam_p)).float().cuda()
    cfg = solver.SolverConfig(max_iters=60)
    got = solver.solve_instances([g.sys], x32, l32, x32, cfg=cfg, fixed_iterations=True,
                                 layout="producer")
    # the same FP32 values, member-major FP64 on the host
    x64 = x32.double().cpu().numpy().transpose(0, 2, 1, 3).copy()
    l64 = l32.double().cpu().numpy().transpose(0, 2, 1, 3).copy()
    ref = solver.solve_instances([g.sys], x64, l64, x64, cfg=cfg, fixed_iterations=True)
    assert np.array_equal(got.xi, ref.xi) and np.array_equal(got.lam, ref.lam)
    # and against the oracle
    xo = np.moveaxis(x64.reshape(B, d.n_d, -1), 0, -1)
    lo = np.moveaxis(l64.reshape(B, d.n_d, -1), 0, -1)
    orc = sf_kron.solve_batch(g.sys, xo, lo, target=xo, max_iters=60, early_exit=False)
    for b in range(B):
        r = np.asarray(orc["xi"][b]).reshape(-1)
        assert np.abs(got.xi[b].reshape(-1) - r).max() / np.abs(r).max() < 1e-9
    # producer layout from host arrays, and a shape error on a member-major tensor
    host = solver.solve_instances([g.sys], prod, lam_p, prod, cfg=cfg, fixed_iterations=True,
                                  layout="producer")
    memb = solver.solve_instances([g.sys], solver.to_member_major(g.xi0, d.n, d.n_basis),
                                  solver.to_member_major(g.lam0, d.n, d.n_basis),
                                  solver.to_member_major(g.xi0, d.n, d.n_basis), cfg=cfg,
                                  fixed_iterations=True)
    assert np.array_equal(host.xi, memb.xi)
    from paper_2510_09204_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        solver.solve_instances([g.sys], torch.zeros((B, d.n_d, d.n, d.n_basis), device="cuda"),
                               None, torch.zeros((B, d.n_d, d.n, d.n_basis), device="cuda"),
                               cfg=cfg, layout="producer")


def test_two_c3_instances_in_one_launch_match_their_reference_goldens():
    """The member -> instance map of a multi-instance launch, pinned to the reference: two C3
    instances (4 samples each, L = 40), members interleaved (instance of member b = b % 2),
    one launch, each member against its own reference solve_batch output."""
    gs = [golden_io.load(f"c3pair_inst{i}_L40") for i in (0, 1)]
    d = gs[0].sys.dims
    mm = [solver.to_member_major(g.xi0, d.n, d.n_basis) for g in gs]
    lm = [solver.to_member_major(g.lam0, d.n, d.n_basis) for g in gs]
    S = mm[0].shape[0]
    order = [(b % 2, b // 2) for b in range(2 * S)]          # (instance, sample) of member b
    xi0 = np.stack([mm[i][s] for i, s in order])
    lam0 = np.stack([lm[i][s] for i, s in order])
    mi = np.array([i for i, _ in order], np.int32)
    cfg = solver.SolverConfig(max_iters=40)
    got = solver.solve_instances([g.sys for g in gs], xi0, lam0, xi0, member_instance=mi, cfg=cfg,
                                 fixed_iterations=True)
    for b, (i, s) in enumerate(order):
        ref = gs[i].out
        r = ref["xi"][s].reshape(-1)
        assert np.abs(got.xi[b].reshape(-1) - r).max() / np.abs(r).max() < 1e-8
        assert np.abs(got.lam[b].reshape(-1) - ref["lam"][s].reshape(-1)).max() < 1e-6
        assert np.abs(got.trace[b][:, 0] - ref["trace"][s][:, 0]).max() < 1e-8
        fr = ref["trace"][s][1:, 1]
        assert np.all(np.abs(got.trace[b][1:, 1] - fr) <= 1e-6 * np.maximum(np.abs(fr), 1e-12))
