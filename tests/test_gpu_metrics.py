"""GPU parity of the post-solve metrics epilogue `sfb_trajectory_metrics`
against the reference's own compute_metrics outputs (tests/golden/metrics_*.npz) and the
metrics oracle; cases mirror the reference's test_metrics.py:23-101."""

import numpy as np
import pytest

from oracle.metrics import trajectory_metrics
from test_oracle import _metrics_cases, load_metrics_golden, metrics_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_09204_b200 import metrics as M  # noqa: E402
from paper_2510_09204_b200.errors import ShapeError  # noqa: E402
from paper_2510_09204_b200.problem import (  # noqa: E402
    BasisConfig, Obstacle, Scenario, ScenarioFamily, build_basis, generate, sample_naive_prior,
    stack_xi, straight_line_coeffs,
)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _golden_batch(name):
    z, nd, obs = load_metrics_golden(name)
    basis = build_basis(BasisConfig(int(z["n_basis"]), int(z["num_steps"]), float(z["duration"])))
    arr = np.stack([np.stack(o) for o in obs]) if obs else None
    mm = np.ascontiguousarray(z["coeffs"].transpose(0, 2, 1, 3))
    return z, basis, arr, mm


@pytest.mark.parametrize("name", _metrics_cases())
def test_metrics_match_reference_golden(name):
    z, basis, arr, mm = _golden_batch(name)
    got = M.metrics_batch(mm, basis, arr, int(z["dense_factor"]))
    for g, m in zip(got, z["metrics"]):
        metrics_close(g, m)


def test_compute_metrics_drop_in_and_per_member_obstacles():
    z, basis, arr, mm = _golden_batch("metrics_d3_moving")
    scn = Scenario(n=6, n_d=3, radii=[0.1] * 3, starts=np.zeros((6, 3)), goals=np.zeros((6, 3)),
                   obstacles=[Obstacle(center=o[0], velocity=o[1], radii=o[2]) for o in arr],
                   p_min=[-2] * 3, p_max=[2] * 3)
    met = M.compute_metrics(z["coeffs"][1], basis, scn)
    metrics_close([getattr(met, f) for f in M.FIELDS], z["metrics"][1])
    assert set(met.to_dict()) >= set(M.FIELDS)
    # per-member obstacle sets: member b sees only obstacle b % 2
    per = np.stack([arr[[b % 2]] for b in range(mm.shape[0])])
    got = M.metrics_batch(mm, basis, per)
    for b in range(mm.shape[0]):
        ref = trajectory_metrics(z["coeffs"][b], 11, 50, 5.0, [tuple(arr[b % 2])], 10)
        metrics_close(got[b], ref)


def test_metrics_c3_batch_against_oracle_and_reproducible():
    cfg = BasisConfig(11, 100, 5.0)
    basis = build_basis(cfg)
    scn = generate(ScenarioFamily("random_box", box=(-2.0, 2.0), n_obstacles=20), 32, 2, seed=7,
                   horizon=cfg)
    xi = stack_xi(sample_naive_prior(scn, basis, 24, seed=7))        # (2, 352, 24)
    mm = np.ascontiguousarray(xi.reshape(2, 32, 11, 24).transpose(3, 0, 1, 2))
    a = M.metrics_batch(mm, basis, scn)
    b = M.metrics_batch(torch.from_numpy(mm).cuda(), basis, scn)
    assert np.array_equal(a, b)
    c = M.metrics_batch(mm[5:9], basis, scn)                       # batch-size independent
    assert np.array_equal(a[5:9], c)
    obs = [(o.center, o.velocity, o.radii) for o in scn.obstacles]
    for k in (0, 3, 23):
        metrics_close(a[k], trajectory_metrics(mm[k].transpose(1, 0, 2), 11, 100, 5.0, obs, 10))


def test_metrics_reference_known_answers():
    """test_metrics.py:23-46, 84-101: stationary robot, straight-line chord, scaled obstacle."""
    basis = build_basis(BasisConfig(11, 50, 5.0))
    still = straight_line_coeffs([[0.3, -0.2]], [[0.3, -0.2]], 11)
    line = straight_line_coeffs([[-1.0, 0.0]], [[1.0, 0.0]], 11)
    obs = Scenario(n=1, n_d=2, radii=[0.1] * 3, starts=[[-0.9, 0.0]], goals=[[-0.9, 0.5]],
                   obstacles=[Obstacle(center=[0.5, 0.0], radii=[0.3] * 3)], p_min=[-1, -1],
                   p_max=[1, 1])
    m0 = M.compute_metrics(still, basis, None)
    assert m0.smoothness < 1e-12 and m0.arc_length < 1e-9 and m0.min_pairwise_clearance == np.inf
    assert abs(M.compute_metrics(line, basis, None).arc_length - 2.0) < 1e-6
    c = straight_line_coeffs(obs.starts, obs.goals, 11)
    m = M.compute_metrics(c, basis, obs)
    pos = M.dense_basis(basis).W @ c[0].T
    expect = np.linalg.norm((pos - [0.5, 0.0]) / 0.3, axis=1).min()
    assert abs(m.min_obstacle_clearance - expect) < 1e-12 and m.min_obstacle_clearance > 1.0


def test_metrics_shape_errors():
    basis = build_basis(BasisConfig(11, 50, 5.0))
    with pytest.raises(ShapeError):
        M.compute_metrics(np.zeros((2, 2, 9)), basis, None)
    with pytest.raises(ShapeError):
        M.metrics_batch(np.zeros((1, 2, 2, 11)), basis, np.zeros((1, 3, 3)))
