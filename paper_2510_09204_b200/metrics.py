"""Post-solve trajectory metrics on the GPU — the drop-in for the reference's
`swarmplan.metrics` (pkg/src/swarmplan/metrics.py:1-87), row f4 of SURVEY.md §8.

`compute_metrics(coeffs, basis, scn, dense_factor)` keeps the reference's signature and
`TrajectoryMetrics` result; `metrics_batch` scores a whole member-major batch in one
`sfb_trajectory_metrics` launch pair (the form the planner's ranking and the benchmark
harness need: pipeline.py:130-133, bench.py:105). There is no CPU path: without the CUDA
library the call raises NativeError.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError
from .problem import BasisConfig, build_basis

FIELDS = ("smoothness", "arc_length", "min_pairwise_clearance", "avg_pairwise_distance",
          "min_obstacle_clearance")


@dataclass
class TrajectoryMetrics:
    """metrics.py:19-37."""

    smoothness: float              # mean ||p_ddot|| over robots and steps, m/s^2
    arc_length: float              # mean per-robot path length, m
    min_pairwise_clearance: float  # m, +inf for a single robot
    avg_pairwise_distance: float
    min_obstacle_clearance: float  # scaled units; >= 1 is collision free
    success: bool | None = None
    iterations: int | None = None

    def to_dict(self) -> dict:
        return {f: getattr(self, f) for f in (*FIELDS, "success", "iterations")}


def dense_basis(basis, factor: int = 10):
    """metrics.py:40-44."""
    cfg = basis.config
    return build_basis(BasisConfig(cfg.n_basis, factor * (cfg.num_steps - 1) + 1, cfg.duration))


def _obstacle_array(obstacles, n_d: int, B: int):
    """(n_obs, 3, n_d) shared or (B, n_obs, 3, n_d) per member from a Scenario, a list of
    Obstacle, or an array; rows are center, velocity, radii[:n_d] (scenario.py:29-44, 99-103)."""
    if obstacles is None:
        return np.zeros((0, 3, n_d)), 0
    if hasattr(obstacles, "obstacles"):
        obstacles = obstacles.obstacles
    if isinstance(obstacles, (list, tuple)):
        if not obstacles:
            return np.zeros((0, 3, n_d)), 0
        arr = np.stack([np.stack([np.asarray(o.center, float)[:n_d],
                                  np.asarray(o.velocity, float)[:n_d],
                                  np.asarray(o.radii, float)[:n_d]]) for o in obstacles])
        return arr, 0
    arr = np.asarray(obstacles, float)
    if arr.ndim == 3 and arr.shape[1:] == (3, n_d):
        return arr, 0
    if arr.ndim == 4 and arr.shape[0] == B and arr.shape[2:] == (3, n_d):
        return arr, arr.shape[1] * 3 * n_d
    raise ShapeError(f"obstacles must be (n_obs, 3, {n_d}) or ({B}, n_obs, 3, {n_d}), got {arr.shape}")


def metrics_batch(coeffs_mm, basis, obstacles=None, dense_factor: int = 10, device=None):
    """Metrics of every member of a batch.

    coeffs_mm: (B, n_d, n, n_basis) member-major coefficients (numpy or CUDA tensor — a
    tensor already on the GPU is used in place, e.g. `DeviceBatch` output).
    Returns a (B, 5) float64 array in FIELDS order."""
    import torch
    if dense_factor < 1:
        raise ShapeError("dense_factor must be >= 1")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    x = coeffs_mm if isinstance(coeffs_mm, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(coeffs_mm, float))
    if x.dim() != 4 or x.shape[3] != basis.config.n_basis:
        raise ShapeError(f"coeffs shape {tuple(x.shape)} incompatible with n_basis={basis.config.n_basis}")
    x = x.to(device=dev, dtype=torch.float64).contiguous()
    B, n_d, n, nb = x.shape
    dense = dense_basis(basis, dense_factor)
    obs, stride = _obstacle_array(obstacles, n_d, B)
    n_obs = obs.shape[-3] if obs.size else 0
    L = _lib.lib()
    nwork = L.sfb_trajectory_metrics_work(B, n_d, n, nb, dense.W.shape[0], n_obs)
    if nwork < 0:
        raise ShapeError("problem shape unsupported by sfb_trajectory_metrics")
    host = [np.ascontiguousarray(a, float).ravel() for a in (basis.Wdd, dense.W, dense.grid, obs)]
    offs = np.cumsum([0] + [a.size for a in host])
    consts = torch.from_numpy(np.concatenate(host)).to(dev)
    scratch = torch.empty(max(int(nwork), 1) + B * 5, dtype=torch.float64, device=dev)
    out = scratch[int(nwork):]
    ptr = lambda k: consts.data_ptr() + 8 * int(offs[k])  # noqa: E731
    s = torch.cuda.current_stream(dev)
    rc = L.sfb_trajectory_metrics(x.data_ptr(), B, n_d, n, nb, ptr(0), basis.Wdd.shape[0], ptr(1),
                                  ptr(2), dense.W.shape[0], ptr(3) if n_obs else None, n_obs, stride,
                                  scratch.data_ptr(), out.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc, "sfb_trajectory_metrics")
    return out.view(B, 5).cpu().numpy()


def compute_metrics(coeffs, basis, scn, dense_factor: int = 10) -> TrajectoryMetrics:
    """metrics.py:48-87: coeffs (n, n_d, n_basis) of one trajectory set."""
    c = np.asarray(coeffs, float)
    if c.ndim != 3 or c.shape[2] != basis.config.n_basis:
        raise ShapeError(f"coeffs shape {c.shape} incompatible with n_basis={basis.config.n_basis}")
    v = metrics_batch(c.transpose(1, 0, 2)[None], basis, scn, dense_factor)[0]
    return TrajectoryMetrics(*map(float, v))
