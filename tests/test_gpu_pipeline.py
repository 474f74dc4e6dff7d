"""GPU parity of the planner stages around the SF: `pipeline.plan`
against the reference's own plan() outputs (tests/golden/plan_*.npz, made by
tests/golden/make_plan_golden.py), and the fused multi-scenario `plan_many`."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2510_09204_b200 import pipeline as P  # noqa: E402
from paper_2510_09204_b200.errors import UsageError  # noqa: E402
from paper_2510_09204_b200.problem import BasisConfig, Obstacle, Scenario  # noqa: E402
from paper_2510_09204_b200.solver import SolverConfig  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ("obs8_default", "obs8_short", "d3_default")


def load(name):
    z = np.load(os.path.join(GOLD, f"plan_{name}.npz"))
    nd = int(z["n_d"])
    hz = z["horizon"]
    obs = [Obstacle(center=o[0, :nd], velocity=o[1, :nd], radii=o[2]) for o in z["obstacles"]]
    scn = Scenario(n=int(z["n"]), n_d=nd, radii=z["radii"], starts=z["starts"], goals=z["goals"],
                   obstacles=obs, p_min=z["p_min"], p_max=z["p_max"],
                   horizon=BasisConfig(int(hz[0]), int(hz[1]), float(hz[2])))
    c = z["cfg"]
    cfg = SolverConfig(rho=c[0], max_iters=int(c[1]), primal_tol=c[2], fp_tol=c[3], d_max=c[4])
    return z, scn, cfg


def test_plan_usage_errors():
    z, scn, cfg = load("obs8_short")
    with pytest.raises(UsageError):
        P.plan(scn, P.CandidateBatch([], "naive_prior"))
    with pytest.raises(UsageError):
        P.plan(scn, P.CandidateBatch(list(z["candidates"][:2]), "naive_prior"), top_k=3)


@pytest.fixture
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_plan_matches_reference(_cuda, name):
    z, scn, cfg = load(name)
    batch = P.CandidateBatch(list(z["candidates"]), "naive_prior")
    res = P.plan(scn, batch, top_k=int(z["top_k"]), cfg=cfg)
    assert np.abs(batch.pre_residual - z["pre"]).max() < 1e-9
    assert np.array_equal(res.order, z["order"])
    assert res.index == int(z["index"]) and res.status == str(z["status"])
    assert [r.iterations for r in res.refined] == list(z["iterations"])
    assert [r.status for r in res.refined] == [str(s) for s in z["statuses"]]
    fin = np.isfinite(z["post"])
    assert np.array_equal(np.isfinite(batch.post_residual), fin)
    assert np.abs(batch.post_residual[fin] - z["post"][fin]).max() < 1e-8
    assert np.abs(batch.smoothness[fin] - z["smooth"][fin]).max() < 1e-8
    assert np.abs(res.coeffs - z["coeffs"]).max() < 1e-8


@pytest.mark.gpu
def test_plan_many_matches_per_scenario_plan(_cuda):
    loaded = [load(n) for n in ("obs8_default", "obs8_short")]
    cfg = loaded[1][2]
    scns = [loaded[0][1], loaded[1][1]]
    cands = [list(l[0]["candidates"]) for l in loaded]
    cands[1] = cands[1][::-1]                    # a different candidate order for scenario 1
    many = P.plan_many(scns, cands, top_k=4, cfg=cfg)
    dev = torch.from_numpy(np.stack([np.stack([c.transpose(1, 0, 2) for c in cs]) for cs in cands])).cuda()
    many_dev = P.plan_many(scns, dev, top_k=4, cfg=cfg)
    for s in range(2):
        one = P.plan(scns[s], P.CandidateBatch(cands[s], "naive_prior"), top_k=4, cfg=cfg)
        for r in (many[s], many_dev[s]):
            assert r.index == one.index and r.status == one.status
            assert np.array_equal(r.order, one.order)
            assert np.abs(r.batch.pre_residual - one.batch.pre_residual).max() < 1e-12
            fin = np.isfinite(one.batch.post_residual)
            assert np.abs(r.batch.post_residual[fin] - one.batch.post_residual[fin]).max() < 1e-12
            assert np.abs(r.batch.smoothness[fin] - one.batch.smoothness[fin]).max() < 1e-12
            assert np.abs(r.coeffs - one.coeffs).max() < 1e-12
