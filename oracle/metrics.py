"""ORACLE (test infrastructure only) — restatement of the reference's post-solve
trajectory metrics, `swarmplan.metrics.compute_metrics` (pkg/src/swarmplan/metrics.py:48-87).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import this
module; the product (`paper_2510_09204_b200.metrics`) runs the CUDA epilogue
`sfb_trajectory_metrics` and never calls into here.

Per trajectory set (coeffs (n, n_d, n_basis)):
  smoothness              mean over robots and basis-grid steps of ||Wdd[k] xi_i||  (:54-55)
  arc_length              mean over robots of sum_k ||p_i(k+1) - p_i(k)|| on the
                          dense grid, dense = factor*(K-1)+1 points              (:57-60)
  min_pairwise_clearance  min over i<j, dense k of ||p_i(k) - p_j(k)|| (inf if n = 1) (:62-67)
  avg_pairwise_distance   mean of the same distances                          (:68)
  min_obstacle_clearance  min over obstacles o, robots, dense k of
                          ||(p_i(k) - c_o - t_k v_o) / r_o[:n_d]|| (inf without obstacles) (:73-78)

Parity status: pinned — `tests/test_oracle.py` checks it against the reference's own
outputs in `tests/golden/metrics_*.npz` (made by tests/golden/make_metrics_golden.py).
"""

from __future__ import annotations

import numpy as np

FIELDS = ("smoothness", "arc_length", "min_pairwise_clearance", "avg_pairwise_distance",
          "min_obstacle_clearance")


def bernstein(n_basis: int, num_steps: int, duration: float):
    """basis.py:62-78: W, Wd, Wdd on a grid of num_steps points over [0, duration]
    (derivatives with respect to time, chain rule 1/T, 1/T^2)."""
    from math import comb
    deg = n_basis - 1
    t = np.linspace(0.0, duration, num_steps)
    s = t / duration

    def B(d, k):
        if k < 0 or k > d:
            return np.zeros_like(s)
        return comb(d, k) * s ** k * (1.0 - s) ** (d - k)

    W = np.stack([B(deg, k) for k in range(n_basis)], axis=1)
    Wd = np.stack([deg * (B(deg - 1, k - 1) - B(deg - 1, k)) for k in range(n_basis)], 1) / duration
    Wdd = np.stack([deg * (deg - 1) * (B(deg - 2, k - 2) - 2 * B(deg - 2, k - 1) + B(deg - 2, k))
                    for k in range(n_basis)], 1) / duration ** 2
    return W, Wd, Wdd, t


def trajectory_metrics(coeffs, n_basis: int, num_steps: int, duration: float, obstacles=(),
                       dense_factor: int = 10) -> np.ndarray:
    """coeffs (n, n_d, n_basis); obstacles: iterable of (center, velocity, radii).
    Returns the five FIELDS as a float64 vector."""
    c = np.asarray(coeffs, float)
    n, n_d, _ = c.shape
    _, _, Wdd, _ = bernstein(n_basis, num_steps, duration)
    Wd_, _, _, td = bernstein(n_basis, dense_factor * (num_steps - 1) + 1, duration)
    acc = np.einsum("kc,ndc->nkd", Wdd, c)
    smooth = float(np.sqrt((acc * acc).sum(axis=2)).mean())
    pos = np.einsum("kc,ndc->nkd", Wd_, c)                    # (n, Kd, n_d)
    seg = np.diff(pos, axis=1)
    arc = float(np.sqrt((seg * seg).sum(axis=2)).sum(axis=1).mean())
    if n >= 2:
        iu, ju = np.triu_indices(n, k=1)
        d = pos[iu] - pos[ju]
        dist = np.sqrt((d * d).sum(axis=2))
        min_clear, avg = float(dist.min()), float(dist.mean())
    else:
        min_clear = avg = float("inf")
    obstacles = list(obstacles)
    if obstacles:
        best = np.inf
        for center, vel, radii in obstacles:
            op = np.asarray(center, float)[None, :] + np.outer(td, np.asarray(vel, float))
            sc = (pos - op[None]) / np.asarray(radii, float)[:n_d]
            best = min(best, float(np.sqrt((sc * sc).sum(axis=2)).min()))
        min_obs = best
    else:
        min_obs = float("inf")
    return np.array([smooth, arc, min_clear, avg, min_obs])
