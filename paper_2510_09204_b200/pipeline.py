"""The planner's three stages around the SF on the GPU: the drop-in for
`swarmplan.pipeline.plan` (pkg/src/swarmplan/pipeline.py:88-153) and a fused
multi-scenario form.

plan(scn, batch, top_k, cfg, sys, basis, warmstarts)
    Same signature, selection rule and result as the reference: rank every candidate by
    its primal residual (stage 1, one zero-iteration launch), refine the top_k in
    projection mode (stage 2, one solve launch), score the refined trajectories'
    smoothness (stage 3, one metrics launch, dense_factor=1) and pick the smoothest
    feasible one — else the lowest post-residual one, flagged infeasible_best_effort.
    Ties break toward the lower candidate index.

plan_many(scenarios, candidates, top_k, cfg, basis)
    I scenarios x C candidates in three launches with no host round trip between the
    stages: residuals, the stable per-scenario argsort and the gather of the top_k
    targets stay on the device; only the final results cross back.

There is no CPU path: every stage runs in libsfb.so (NativeError without it).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

from . import solver as S
from .errors import UsageError
from .metrics import metrics_batch
from .problem import assemble, build_basis, stack_xi
from .problem import sample_naive_prior as _naive_list

DEFAULT_COUNT = 256      # pipeline.py:27
DEFAULT_TOP_K = 10       # pipeline.py:28


@dataclass
class CandidateBatch:
    """pipeline.py:32-41."""

    candidates: list
    source: str
    pre_residual: np.ndarray | None = None
    post_residual: np.ndarray | None = None
    smoothness: np.ndarray | None = None

    def __len__(self) -> int:
        return len(self.candidates)


@dataclass
class PlanResult:
    """pipeline.py:44-56."""

    coeffs: np.ndarray
    index: int
    status: str
    batch: CandidateBatch
    order: np.ndarray
    refined: list
    smoothness: float

    @property
    def best_refined(self):
        return self.refined[int(np.flatnonzero(self.order == self.index)[0])]


def sample_naive_prior(scn, basis, count: int, seed: int = 0, noise_scale: float | None = None):
    """pipeline.py:59-82, returning a CandidateBatch."""
    return CandidateBatch(candidates=_naive_list(scn, basis, count, seed=seed, noise_scale=noise_scale),
                          source="naive_prior")


def _select(top, post, smooth, primal_tol):
    """pipeline.py:137-143."""
    feasible = [int(i) for i in top if post[i] < primal_tol]
    if feasible:
        return min(feasible, key=lambda i: (smooth[i], i)), "success"
    return min((int(i) for i in top), key=lambda i: (post[i], i)), "infeasible_best_effort"


def plan(scn, batch: CandidateBatch, top_k: int = DEFAULT_TOP_K, cfg=None, sys=None, basis=None,
         warmstarts=None) -> PlanResult:
    """pipeline.py:88-153 with every numeric stage on the GPU."""
    if len(batch) == 0:
        raise UsageError("candidate batch is empty")
    if top_k > len(batch):
        raise UsageError(f"top_k ({top_k}) exceeds batch size ({len(batch)})")
    cfg = cfg or S.SolverConfig()
    if basis is None:
        basis = build_basis(scn.horizon)
    sys = sys or assemble(scn, basis, d_max=cfg.d_max)
    xi_all = stack_xi(batch.candidates)
    batch.pre_residual = S.batch_primal_residual(xi_all, sys)
    order = np.argsort(batch.pre_residual, kind="stable")
    top = order[:top_k]
    targets = xi_all[..., top]
    mode = S.ObjectiveMode.projection(targets)
    if warmstarts is not None:
        xi0 = stack_xi([warmstarts[i][0] for i in top])
        lam0 = stack_xi([warmstarts[i][1] for i in top])
    else:
        xi0, lam0 = targets.copy(), np.zeros_like(targets)
    cache = S.KktCache(sys, mode, cfg)
    refined = S.solve_batch(S.SolverState(xi=xi0, lam=lam0), sys, mode, cfg, cache)
    d = sys.dims
    post = np.full(len(batch), np.nan)
    smooth = np.full(len(batch), np.nan)
    mm = np.stack([r.xi.reshape(d.n_d, d.n, d.n_basis) for r in refined])
    sm = metrics_batch(mm, basis, scn, dense_factor=1)[:, 0]
    for pos, idx in enumerate(top):
        post[idx] = refined[pos].primal
        smooth[idx] = sm[pos]
    batch.post_residual, batch.smoothness = post, smooth
    best, status = _select(top, post, smooth, cfg.primal_tol)
    best_pos = int(np.flatnonzero(top == best)[0])
    return PlanResult(coeffs=refined[best_pos].coeffs(sys), index=int(best), status=status,
                      batch=batch, order=order, refined=refined, smoothness=float(smooth[best]))


def _obstacles(scn, n_d):
    if not scn.obstacles:
        return np.zeros((0, 3, n_d))
    return np.stack([np.stack([np.asarray(o.center, float)[:n_d], np.asarray(o.velocity, float)[:n_d],
                               np.asarray(o.radii, float)[:n_d]]) for o in scn.obstacles])


def plan_many(scenarios, candidates, top_k: int = DEFAULT_TOP_K, cfg=None, basis=None,
              device=None, cluster: int = 0) -> list[PlanResult]:
    """Plan I scenarios at once. `candidates`: per scenario a CandidateBatch or a list of
    (n, n_d, n_basis) arrays (same count C for every scenario), or a CUDA tensor
    (I, C, n_d, n, n_basis) in member-major layout (e.g. straight from a sampler) that is
    used in place. All scenarios must share n, n_d, the horizon and the obstacle count."""
    import torch
    cfg = cfg or S.SolverConfig()
    I = len(scenarios)
    if I == 0:
        raise UsageError("no scenarios")
    if basis is None:
        basis = build_basis(scenarios[0].horizon)
    systems = [assemble(s, basis, d_max=cfg.d_max) for s in scenarios]
    d = systems[0].dims
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if isinstance(candidates, torch.Tensor):
        cand = candidates.to(device=dev, dtype=torch.float64)
        if cand.dim() != 5 or cand.shape[0] != I:
            raise UsageError("candidate tensor must be (I, C, n_d, n, n_basis)")
        lists = None
    else:
        lists = [c.candidates if isinstance(c, CandidateBatch) else list(c) for c in candidates]
        if len(lists) != I or len({len(c) for c in lists}) != 1:
            raise UsageError("every scenario needs the same number of candidates")
        host = np.stack([np.stack([np.asarray(x, float).transpose(1, 0, 2) for x in c]) for c in lists])
        cand = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
    C = cand.shape[1]
    if C == 0:
        raise UsageError("candidate batch is empty")
    if top_k > C:
        raise UsageError(f"top_k ({top_k}) exceeds batch size ({C})")
    flat = cand.reshape(I * C, d.n_d, d.n, d.n_basis).contiguous()
    # stage 1: primal residual of every candidate (pipeline.py:113-115)
    zero = dataclasses.replace(cfg, max_iters=0) if dataclasses.is_dataclass(cfg) else \
        S.SolverConfig(rho=cfg.rho, max_iters=0, primal_tol=cfg.primal_tol, fp_tol=cfg.fp_tol, d_max=cfg.d_max)
    mi1 = np.repeat(np.arange(I, dtype=np.int32), C)
    rank = S.DeviceBatch(systems, flat, None, flat, cfg=zero, member_instance=mi1, early_exit=False,
                         trace=False, device=dev.index, cluster=cluster)
    rank.launch()
    pre = rank.out_primal.view(I, C)
    order = torch.argsort(pre, dim=1, stable=True)
    top = order[:, :top_k]
    sel = (torch.arange(I, device=dev)[:, None] * C + top).reshape(-1)
    targets = flat.index_select(0, sel).contiguous()
    # stage 2: refine the top_k of every scenario in one launch (pipeline.py:117-126)
    mi2 = np.repeat(np.arange(I, dtype=np.int32), top_k)
    ref = S.DeviceBatch(systems, targets, None, targets, cfg=cfg, member_instance=mi2, early_exit=True,
                        trace=True, device=dev.index, cluster=cluster)
    ref.launch()
    # stage 3: smoothness of the refined trajectories (pipeline.py:130-133, dense_factor = 1)
    obs = np.stack([_obstacles(s, d.n_d) for s in scenarios])[mi2]
    sm = metrics_batch(ref.out_xi, basis, obs, dense_factor=1, device=dev.index)[:, 0]
    out = ref.results()
    pre_h, order_h = pre.cpu().numpy(), order.cpu().numpy()
    results = []
    for s in range(I):
        refined = []
        for p in range(top_k):
            b = s * top_k + p
            refined.append(S.SolverResult(
                xi=out["xi"][b].reshape(d.n_d, d.nvar_ax), lam=out["lam"][b].reshape(d.n_d, d.nvar_ax),
                status=out["status"][b], iterations=int(out["iterations"][b]),
                primal=float(out["primal"][b]), trace=out["trace"][b],
                eq_violation_max=float(out["eq_max"][b])))
        tk = order_h[s, :top_k]
        post, smooth = np.full(C, np.nan), np.full(C, np.nan)
        post[tk] = out["primal"][s * top_k:(s + 1) * top_k]
        smooth[tk] = sm[s * top_k:(s + 1) * top_k]
        if lists is not None and isinstance(candidates[s], CandidateBatch):
            batch = candidates[s]
        else:
            batch = CandidateBatch(candidates=lists[s] if lists is not None else
                                   [x.cpu().numpy().transpose(1, 0, 2) for x in cand[s]], source="device")
        batch.pre_residual, batch.post_residual, batch.smoothness = pre_h[s].copy(), post, smooth
        best, status = _select(tk, post, smooth, cfg.primal_tol)
        best_pos = int(np.flatnonzero(tk == best)[0])
        results.append(PlanResult(coeffs=refined[best_pos].coeffs(systems[s]), index=int(best),
                                  status=status, batch=batch, order=order_h[s].copy(), refined=refined,
                                  smoothness=float(smooth[best])))
    return results
