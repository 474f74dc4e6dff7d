"""Host-side problem model feeding the SF solver: Bernstein basis, scenarios and
the per-instance constraint data.

This is input plumbing, not the hot path. It exists so the drop-in can build
inputs on machines where the reference package is absent (the GPU box) while
producing the same numbers the reference would:

* `build_basis` restates `pkg/src/swarmplan/basis.py:45-78` (Bernstein W, Wd,
  Wdd on a uniform grid of `num_steps` points over [0, duration]).
* `generate` restates the random-box / antipodal-circle generators of
  `pkg/src/swarmplan/scenario.py:116-188` with the same RNG call sequence, so a
  seed yields the reference's scenario bit for bit (checked in
  `tests/test_host.py:82-108` against the reference in the dev container).
* `assemble` restates the parts of `pkg/src/swarmplan/constraints.py:95-156`
  the B200 solver needs: the boundary matrix A = I_n (x) E and b, the workspace
  bounds h, the obstacle trajectories and the inflated contact axes. The dense
  selection matrix F and box matrix G are never built (they are implied by the
  structure; `oracle/sf_dense.py` builds them when it needs them).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import comb

import numpy as np

from .errors import ConfigError, GenerationError, ShapeError, ValidationError

DEFAULT_MARGIN = 1.1          # constraints.py:27
PLACEMENT_MARGIN = 1.15       # scenario.py:25
_MAX_TRIES = 5000             # scenario.py:26
NOISE_FRACTION = 0.25         # pipeline.py:29


# --------------------------------------------------------------------------- basis
@dataclass(frozen=True)
class BasisConfig:
    """basis.py:19-33: degree n_basis-1 Bernstein basis on num_steps grid points."""

    n_basis: int = 11
    num_steps: int = 50
    duration: float = 5.0

    def __post_init__(self):
        if self.n_basis < 4:
            raise ConfigError(f"n_basis must be >= 4, got {self.n_basis}")
        if self.num_steps < self.n_basis:
            raise ConfigError(
                f"num_steps ({self.num_steps}) must be >= n_basis ({self.n_basis})")
        if not self.duration > 0:
            raise ConfigError(f"duration must be > 0, got {self.duration}")


@dataclass(frozen=True)
class BasisMatrices:
    W: np.ndarray     # (K+1, n_basis)
    Wd: np.ndarray
    Wdd: np.ndarray
    grid: np.ndarray  # (K+1,)
    config: BasisConfig


def _bernstein(degree: int, tau: np.ndarray) -> np.ndarray:
    tau = np.asarray(tau, dtype=float)[:, None]
    j = np.arange(degree + 1)[None, :]
    coef = np.array([float(comb(degree, int(x))) for x in range(degree + 1)])[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        out = coef * tau**j * (1.0 - tau) ** (degree - j)
    return np.nan_to_num(out, nan=1.0)


def _shift(mat: np.ndarray, offset: int, total: int) -> np.ndarray:
    out = np.zeros((mat.shape[0], total))
    out[:, offset: offset + mat.shape[1]] = mat
    return out


def build_basis(cfg: BasisConfig) -> BasisMatrices:
    """basis.py:62-78."""
    deg = cfg.n_basis - 1
    grid = np.linspace(0.0, cfg.duration, cfg.num_steps)
    tau = grid / cfg.duration
    W = _bernstein(deg, tau)
    b1 = _bernstein(deg - 1, tau)
    Wd = deg * (_shift(b1, 1, deg + 1) - _shift(b1, 0, deg + 1)) / cfg.duration
    b2 = _bernstein(deg - 2, tau)
    Wdd = deg * (deg - 1) * (
        _shift(b2, 2, deg + 1) - 2.0 * _shift(b2, 1, deg + 1) + _shift(b2, 0, deg + 1)
    ) / cfg.duration**2
    return BasisMatrices(W=W, Wd=Wd, Wdd=Wdd, grid=grid, config=cfg)


def straight_line_coeffs(starts, goals, n_basis: int) -> np.ndarray:
    """basis.py:110-116: control points on the start->goal segment."""
    starts = np.asarray(starts, dtype=float)
    goals = np.asarray(goals, dtype=float)
    frac = np.linspace(0.0, 1.0, n_basis)
    return starts[:, :, None] + (goals - starts)[:, :, None] * frac[None, None, :]


# ------------------------------------------------------------------------ scenario
@dataclass
class Obstacle:
    """scenario.py:29-44."""

    center: np.ndarray
    radii: np.ndarray
    velocity: np.ndarray | None = None

    def __post_init__(self):
        self.center = np.asarray(self.center, dtype=float)
        self.radii = np.asarray(self.radii, dtype=float)
        self.velocity = (np.zeros_like(self.center) if self.velocity is None
                         else np.asarray(self.velocity, dtype=float))


@dataclass
class Scenario:
    """scenario.py:47-103 (data model + validate + obstacle trajectories)."""

    n: int
    n_d: int
    radii: np.ndarray
    starts: np.ndarray
    goals: np.ndarray
    obstacles: list
    p_min: np.ndarray
    p_max: np.ndarray
    horizon: BasisConfig = field(default_factory=BasisConfig)
    seed: int = 0

    def __post_init__(self):
        self.radii = np.asarray(self.radii, dtype=float)
        self.starts = np.asarray(self.starts, dtype=float)
        self.goals = np.asarray(self.goals, dtype=float)
        self.p_min = np.asarray(self.p_min, dtype=float)
        self.p_max = np.asarray(self.p_max, dtype=float)

    @property
    def contact_distance(self) -> float:
        return 2.0 * float(self.radii[0])

    @property
    def contact_axes(self) -> np.ndarray:
        return 2.0 * self.radii

    def validate(self) -> None:
        if self.n_d not in (2, 3):
            raise ValidationError(f"n_d must be 2 or 3, got {self.n_d}")
        for name, arr in (("starts", self.starts), ("goals", self.goals)):
            if arr.shape != (self.n, self.n_d):
                raise ValidationError(f"{name} must have shape ({self.n}, {self.n_d})")
            if not np.isfinite(arr).all():
                raise ValidationError(f"{name} contains non-finite values")
            if ((arr < self.p_min) | (arr > self.p_max)).any():
                raise ValidationError(f"{name} outside workspace box")
        a = self.contact_distance
        for name, arr in (("starts", self.starts), ("goals", self.goals)):
            if self.n >= 2:
                d = np.linalg.norm(arr[:, None] - arr[None, :], axis=2)
                d[np.diag_indices(self.n)] = np.inf
                if d.min() < a:
                    raise ValidationError(f"{name} pairwise separation below contact distance")
            for obs in self.obstacles:
                scaled = (arr - obs.center) / obs.radii[: self.n_d]
                if (np.linalg.norm(scaled, axis=1) < 1.0).any():
                    raise ValidationError(f"{name} inside an inflated obstacle")

    def obstacle_positions(self, grid: np.ndarray) -> np.ndarray:
        """(n_obs, K+1, n_d), scenario.py:99-103."""
        if not self.obstacles:
            return np.zeros((0, len(grid), self.n_d))
        return np.stack([o.center + np.outer(grid, o.velocity) for o in self.obstacles])


@dataclass(frozen=True)
class ScenarioFamily:
    """scenario.py:106-113."""

    kind: str
    robot_radius: float = 0.1
    box: tuple = (-1.0, 1.0)
    circle_radius: float = 1.0
    n_obstacles: int = 0
    obstacle_radius: float = 0.15


def _place(rng, count, n_d, lo, hi, min_sep, obstacles, what):
    """Rejection sampling with the reference's draw order (scenario.py:116-134)."""
    pts: list[np.ndarray] = []
    for _ in range(count):
        for _try in range(_MAX_TRIES):
            p = rng.uniform(lo, hi, size=n_d)
            if any(np.linalg.norm(p - q) < min_sep for q in pts):
                continue
            if any(np.linalg.norm((p - o.center) / (PLACEMENT_MARGIN * o.radii[:n_d])) < 1.0
                   for o in obstacles):
                continue
            pts.append(p)
            break
        else:
            raise GenerationError(
                f"could not place {what} point {len(pts)} with separation {min_sep}")
    return np.array(pts)


def generate(family: ScenarioFamily, n: int, n_d: int = 2, seed: int = 0,
             horizon: BasisConfig | None = None) -> Scenario:
    """scenario.py:137-188; deterministic for (family, n, n_d, seed)."""
    if n < 1:
        raise GenerationError("need at least one robot")
    horizon = horizon or BasisConfig()
    rng = np.random.default_rng(seed)
    r = family.robot_radius
    radii = np.array([r, r, r])
    min_sep = PLACEMENT_MARGIN * 2.0 * r
    if family.kind == "random_box":
        lo, hi = family.box
        obstacles = []
        for _ in range(family.n_obstacles):
            size = family.obstacle_radius + r
            c = rng.uniform(lo + size, hi - size, size=n_d)
            obstacles.append(Obstacle(center=c, radii=np.full(3, size)))
        starts = _place(rng, n, n_d, lo + r, hi - r, min_sep, obstacles, "start")
        goals = _place(rng, n, n_d, lo + r, hi - r, min_sep, obstacles, "goal")
        p_min, p_max = np.full(n_d, lo), np.full(n_d, hi)
    elif family.kind == "circle_antipodal":
        R = family.circle_radius
        if n >= 2 and 2.0 * R * np.sin(np.pi / n) < min_sep:
            raise GenerationError(
                f"{n} robots on a circle of radius {R} violate the separation constraint")
        ang = 2.0 * np.pi * np.arange(n) / n
        starts = np.zeros((n, n_d))
        starts[:, 0] = R * np.cos(ang)
        starts[:, 1] = R * np.sin(ang)
        goals = -starts
        obstacles = []
        ext = 1.25 * R + 2.0 * r
        p_min, p_max = np.full(n_d, -ext), np.full(n_d, ext)
    else:
        raise GenerationError(f"unknown scenario family {family.kind!r}")
    scn = Scenario(n=n, n_d=n_d, radii=radii, starts=starts, goals=goals,
                   obstacles=obstacles, p_min=p_min, p_max=p_max, horizon=horizon, seed=seed)
    scn.validate()
    return scn


def sample_naive_prior(scn: Scenario, basis: BasisMatrices, count: int, seed: int = 0,
                       noise_scale: float | None = None) -> list[np.ndarray]:
    """pipeline.py:59-82: straight line + N(0, sigma) on interior coefficients.

    Stand-in for flow samples; returns the candidate list only."""
    from .errors import UsageError
    if count < 1:
        raise UsageError("count must be >= 1")
    if noise_scale is None:
        noise_scale = NOISE_FRACTION * float((scn.p_max - scn.p_min).max())
    rng = np.random.default_rng(seed)
    base = straight_line_coeffs(scn.starts, scn.goals, basis.config.n_basis)
    cands = [base.copy()]
    for _ in range(count - 1):
        noise = np.zeros_like(base)
        noise[:, :, 1:-1] = noise_scale * rng.standard_normal(base[:, :, 1:-1].shape)
        cands.append(base + noise)
    return cands


# ---------------------------------------------------------------------- assembly
@dataclass(frozen=True)
class SystemDims:
    """constraints.py:30-50 (same field names)."""

    n: int
    n_d: int
    n_basis: int
    num_steps: int
    n_obs: int
    n_pairs: int
    rows_pairs: int
    rows_obs: int
    nvar_ax: int
    a_rows: int
    g_rows: int

    @property
    def f_rows(self) -> int:
        return self.rows_pairs + self.rows_obs

    @property
    def nvar(self) -> int:
        return self.n_d * self.nvar_ax


@dataclass(frozen=True)
class ConstraintSystem:
    """Structured counterpart of constraints.py:53-67.

    Carries the same fields except the dense F and G, which are `None` here:
    they are fully determined by (n, n_obs, W) and the B200 solver never needs
    them. A reference `ConstraintSystem` (with dense F, G) is accepted by the
    solver too; only the fields below are read."""

    A: np.ndarray          # (a_rows, nvar_ax) = I_n (x) E
    b: np.ndarray          # (n_d, a_rows)
    h: np.ndarray          # (n_d, g_rows) = [p_max..., -p_min...] per axis
    pair_axes: np.ndarray  # (3,) = margin * 2 * radii
    obs_axes: np.ndarray   # (n_obs, 3)
    obs_pos: np.ndarray    # (n_d, n_obs, K+1)
    dims: SystemDims
    basis: BasisMatrices
    d_max: float = 1e6
    F: np.ndarray | None = None
    G: np.ndarray | None = None


def boundary_rows(basis: BasisMatrices, rest_to_rest: bool = True) -> np.ndarray:
    """E of constraints.py:111-114: W0, WK (+ Wd0, WdK, Wdd0, WddK)."""
    rows = [basis.W[0], basis.W[-1]]
    if rest_to_rest:
        rows += [basis.Wd[0], basis.Wd[-1], basis.Wdd[0], basis.Wdd[-1]]
    return np.stack(rows)


def assemble(scn: Scenario, basis: BasisMatrices, margin: float = DEFAULT_MARGIN,
             rest_to_rest: bool = True, d_max: float = 1e6) -> ConstraintSystem:
    """constraints.py:95-156 without the dense F/G."""
    if basis.config != scn.horizon:
        raise ShapeError("basis does not match the scenario horizon")
    n, n_d, n_xi = scn.n, scn.n_d, basis.config.n_basis
    K1 = basis.config.num_steps
    n_obs = len(scn.obstacles)
    E = boundary_rows(basis, rest_to_rest)
    nb = E.shape[0]
    A = np.kron(np.eye(n), E)
    b = np.zeros((n_d, A.shape[0]))
    for ax in range(n_d):
        for i in range(n):
            b[ax, i * nb] = scn.starts[i, ax]
            b[ax, i * nb + 1] = scn.goals[i, ax]
    h = np.zeros((n_d, 2 * n * K1))
    for ax in range(n_d):
        h[ax, : n * K1] = scn.p_max[ax]
        h[ax, n * K1:] = -scn.p_min[ax]
    obs_axes = (margin * np.stack([o.radii for o in scn.obstacles]) if n_obs
                else np.zeros((0, 3)))
    obs_pos = scn.obstacle_positions(basis.grid).transpose(2, 0, 1)
    n_pairs = n * (n - 1) // 2
    dims = SystemDims(n=n, n_d=n_d, n_basis=n_xi, num_steps=K1, n_obs=n_obs,
                      n_pairs=n_pairs, rows_pairs=n_pairs * K1, rows_obs=n * n_obs * K1,
                      nvar_ax=n * n_xi, a_rows=A.shape[0], g_rows=2 * n * K1)
    return ConstraintSystem(A=A, b=b, h=h, pair_axes=margin * scn.contact_axes,
                            obs_axes=obs_axes, obs_pos=np.ascontiguousarray(obs_pos),
                            dims=dims, basis=basis, d_max=d_max)


def xi_from_coeffs(coeffs) -> np.ndarray:
    """solver.py:132-136: (n, n_d, n_basis) -> (n_d, nvar_ax, 1)."""
    coeffs = np.asarray(coeffs, dtype=float)
    n, n_d, n_xi = coeffs.shape
    return coeffs.transpose(1, 0, 2).reshape(n_d, n * n_xi, 1)


def stack_xi(coeff_list) -> np.ndarray:
    """solver.py:139-141."""
    return np.concatenate([xi_from_coeffs(c) for c in coeff_list], axis=-1)
