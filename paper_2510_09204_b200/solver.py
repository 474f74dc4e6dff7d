"""Drop-in for the reference SF entry point `swarmplan.solver` on B200.

Same public names, signatures, argument meaning, result fields and error types as
`pkg/src/swarmplan/solver.py` (SolverConfig :29-41, ObjectiveMode :44-61,
KktCache :64-91, SolverState/SolverResult :94-129, fixed_point_step :246-256,
solve_batch :286-355, solve :358-367). Every map evaluation runs in the sm_100a
kernel behind `libsfb.so` (include/sfb.h); this module only validates inputs,
converts layouts and moves buffers. There is no CPU fallback.

Beyond the reference API, `solve_instances` solves many instances x samples in
one launch (the north-star batch shape; the reference takes a single system per
call) and `DeviceBatch` keeps a prepared batch resident on the GPU for repeated
solves (benchmarking, serving).
"""

from __future__ import annotations

import ctypes
import hashlib
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import SetupError, ShapeError, UsageError

# --------------------------------------------------------------------------- types


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:29-41."""

    rho: float = 1.0
    max_iters: int = 15000
    primal_tol: float = 1e-3
    fp_tol: float = 1e-8
    d_max: float = 1e6

    def __post_init__(self):
        if not self.rho > 0:
            raise SetupError(f"rho must be positive, got {self.rho}")
        if not (self.primal_tol > 0 and self.fp_tol > 0):
            raise SetupError("tolerances must be positive")


@dataclass(frozen=True)
class ObjectiveMode:
    """solver.py:44-61."""

    kind: str
    target: np.ndarray | None = None

    @classmethod
    def projection(cls, target) -> "ObjectiveMode":
        return cls(kind="projection", target=np.asarray(target, dtype=float))

    @classmethod
    def smoothness(cls) -> "ObjectiveMode":
        return cls(kind="smoothness")


@dataclass
class SolverState:
    """solver.py:94-105: batched iterate, trailing batch axis."""

    xi: np.ndarray
    lam: np.ndarray
    s: np.ndarray | None = None
    vars: object | None = None
    iteration: int = 0

    @property
    def batch_size(self) -> int:
        return self.xi.shape[-1]


@dataclass
class SolverResult:
    """solver.py:108-129."""

    xi: np.ndarray
    lam: np.ndarray
    status: str
    iterations: int
    primal: float
    trace: np.ndarray
    eq_violation_max: float
    wall_time: float = 0.0

    @property
    def success(self) -> bool:
        return self.status == "converged_primal"

    def coeffs(self, sys) -> np.ndarray:
        d = sys.dims
        return self.xi.reshape(d.n_d, d.n, d.n_basis).transpose(1, 0, 2)

    def iterations_to(self, threshold: float) -> int | None:
        below = np.flatnonzero(self.trace[:, 0] < threshold)
        return int(below[0]) if below.size else None


# ------------------------------------------------------------------ system data


@dataclass
class SystemData:
    """What the kernel reads from one ConstraintSystem (constraints.py:53-67)."""

    n: int
    n_d: int
    n_basis: int
    num_steps: int
    n_obs: int
    n_bnd: int
    W: np.ndarray
    Wdd: np.ndarray
    E: np.ndarray
    bvals: np.ndarray      # (n_d, n, n_bnd)
    box: np.ndarray        # (2, n_d): p_min, p_max
    obs_pos: np.ndarray    # (n_d, m, K1)
    obs_axes: np.ndarray   # (m, 3)
    pair_axes: np.ndarray  # (3,)
    d_max: float

    @property
    def shape_key(self):
        return (self.n, self.n_d, self.n_basis, self.num_steps, self.n_obs, self.n_bnd)


def _dense_kkt_cond(sys, kind: str, rho: float) -> float:
    """cond(M) of the reference KKT matrix (solver.py:68-83), used only to classify a
    constraint system that is not Kronecker-structured (setup time, host)."""
    d = sys.dims
    F = getattr(sys, "F", None)
    G = getattr(sys, "G", None)
    W = np.asarray(sys.basis.W, float)
    if F is None or G is None:
        pairs = [(i, j) for i in range(d.n) for j in range(i + 1, d.n)]
        D = np.zeros((len(pairs), d.n))
        for r, (i, j) in enumerate(pairs):
            D[r, i], D[r, j] = 1.0, -1.0
        blocks = [np.kron(D, W)] if pairs else []
        if d.n_obs:
            blocks.append(np.kron(np.eye(d.n), np.kron(np.ones((d.n_obs, 1)), W)))
        F = np.vstack(blocks) if blocks else np.zeros((0, d.n * d.n_basis))
        pos = np.kron(np.eye(d.n), W)
        G = np.vstack([pos, -pos])
    nv = d.nvar_ax
    Q = np.eye(nv) if kind == "projection" else np.kron(np.eye(d.n), sys.basis.Wdd.T @ sys.basis.Wdd)
    H = Q + rho * (F.T @ F + G.T @ G)
    A = np.asarray(sys.A, float)
    M = np.zeros((nv + A.shape[0],) * 2)
    M[:nv, :nv] = H
    M[:nv, nv:] = A.T
    M[nv:, :nv] = A
    return float(np.linalg.cond(M))


def system_data(sys, kind: str = "projection", rho: float = 1.0) -> SystemData:
    """Extract and validate the structured data of a (reference or local) ConstraintSystem."""
    d = sys.dims
    n, n_d, n_xi, K1, m = d.n, d.n_d, d.n_basis, d.num_steps, d.n_obs
    A = np.asarray(sys.A, float)
    if A.shape[1] != n * n_xi or A.shape[0] % n != 0:
        if _dense_kkt_cond(sys, kind, rho) > 1e14:
            raise SetupError("KKT matrix is singular or near-singular")
        raise UsageError("boundary matrix A is not I_n (x) E: unsupported constraint system")
    nb = A.shape[0] // n
    E = A[:nb, :n_xi].copy()
    if not np.array_equal(A, np.kron(np.eye(n), E)):
        if _dense_kkt_cond(sys, kind, rho) > 1e14:
            raise SetupError("KKT matrix is singular or near-singular")
        raise UsageError("boundary matrix A is not I_n (x) E: unsupported constraint system")
    b = np.asarray(sys.b, float)
    if b.shape != (n_d, n * nb):
        raise ShapeError(f"b has shape {b.shape}, expected {(n_d, n * nb)}")
    h = np.asarray(sys.h, float)
    if h.shape != (n_d, 2 * n * K1):
        raise ShapeError(f"h has shape {h.shape}, expected {(n_d, 2 * n * K1)}")
    pmax, pmin = h[:, 0].copy(), -h[:, n * K1].copy()
    if not (np.all(h[:, : n * K1] == pmax[:, None]) and np.all(-h[:, n * K1:] == pmin[:, None])):
        raise UsageError("workspace bounds h are not a per-axis box: unsupported constraint system")
    obs_pos = np.asarray(sys.obs_pos, float).reshape(n_d, m, K1)
    obs_axes = np.asarray(sys.obs_axes, float).reshape(m, 3)
    W = np.ascontiguousarray(np.asarray(sys.basis.W, float))
    if W.shape != (K1, n_xi):
        raise ShapeError(f"basis W has shape {W.shape}, expected {(K1, n_xi)}")
    return SystemData(n=n, n_d=n_d, n_basis=n_xi, num_steps=K1, n_obs=m, n_bnd=nb, W=W,
                      Wdd=np.ascontiguousarray(np.asarray(sys.basis.Wdd, float)),
                      E=np.ascontiguousarray(E), bvals=np.ascontiguousarray(b.reshape(n_d, n, nb)),
                      box=np.stack([pmin, pmax]), obs_pos=np.ascontiguousarray(obs_pos),
                      obs_axes=np.ascontiguousarray(obs_axes),
                      pair_axes=np.asarray(sys.pair_axes, float).reshape(3).copy(),
                      d_max=float(sys.d_max))


# ------------------------------------------------------------------------- plan


class Plan:
    """Owns one `sfb_plan` (the Kronecker KKT inverse on the device)."""

    def __init__(self, sd: SystemData, kind: str, rho: float, device: int):
        L = _lib.lib()
        if kind not in _lib.MODE:
            raise UsageError(f"unknown objective kind {kind!r}")
        self.kind, self.rho, self.device = kind, float(rho), device
        self.shape_key = sd.shape_key
        dims = _lib.Dims(sd.n, sd.n_d, sd.n_basis, sd.num_steps, sd.n_obs, sd.n_bnd)
        ptr = ctypes.c_void_p()
        import torch
        with torch.cuda.device(device):
            rc = L.sfb_plan_create(ctypes.byref(ptr), ctypes.byref(dims),
                                   sd.W.ctypes.data, sd.Wdd.ctypes.data, sd.E.ctypes.data,
                                   float(rho), _lib.MODE[kind])
        _lib.check(rc, "sfb_plan_create")
        self._ptr = ptr
        self.cond = L.sfb_plan_cond(ptr)
        self.smem_bytes = int(L.sfb_smem_bytes(ptr))

    @property
    def handle(self):
        return self._ptr

    def __del__(self):
        ptr = getattr(self, "_ptr", None)
        L = getattr(_lib, "_LIB", None) if _lib is not None else None
        if ptr is not None and ptr.value and L is not None:
            L.sfb_plan_destroy(ptr)
            self._ptr = None


_PLANS: dict = {}


def get_plan(sd: SystemData, kind: str, rho: float, device: int | None = None) -> Plan:
    """Plans are instance-independent: one per (shape, basis, E, rho, mode)."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    h = hashlib.sha1()
    for arr in (sd.W, sd.E, sd.Wdd if kind == "smoothness" else np.zeros(0)):
        h.update(np.ascontiguousarray(arr).tobytes())
    key = (sd.shape_key, kind, float(rho), device, h.hexdigest())
    plan = _PLANS.get(key)
    if plan is None:
        plan = Plan(sd, kind, rho, device)
        if len(_PLANS) > 64:
            _PLANS.clear()
        _PLANS[key] = plan
    return plan


class KktCache:
    """Drop-in for solver.py:64-91: validates the system, checks cond(M) and holds the plan."""

    def __init__(self, sys, mode, cfg):
        kind = getattr(mode, "kind", mode)
        if kind not in ("projection", "smoothness"):
            raise UsageError(f"unknown objective kind {kind!r}")
        sd = system_data(sys, kind, cfg.rho)
        self.plan = get_plan(sd, kind, cfg.rho)
        self.size = sys.dims.nvar_ax + sd.n * sd.n_bnd
        self.nvar_ax = sys.dims.nvar_ax
        self.kind = kind
        self.rho = float(cfg.rho)
        self.cond = self.plan.cond


# ---------------------------------------------------------------- device batch


def _as_tensor(x, device, dtype, counter=None):
    import torch
    if isinstance(x, torch.Tensor):
        if counter is not None and x.device.type == "cpu":
            counter[0] += x.numel() * torch.empty(0, dtype=dtype).element_size()
        return x.to(device=device, dtype=dtype).contiguous()
    t = torch.as_tensor(np.ascontiguousarray(x), dtype=dtype)
    if counter is not None:
        counter[0] += t.numel() * t.element_size()
    return t.to(device)


class DeviceBatch:
    """A batch of members (instance x sample) resident on one GPU.

    Inputs are member-major: xi0/lam0/target (B, n_d, n, n_basis). `systems` is one
    constraint system per instance (all with the same shape and basis);
    member_instance[b] selects member b's instance."""

    def __init__(self, systems, xi0, lam0=None, target=None, kind="projection", cfg=None,
                 member_instance=None, early_exit=True, trace=True, counters=False,
                 device=None, cluster=0):
        import torch
        cfg = cfg or SolverConfig()
        if not isinstance(systems, (list, tuple)):
            systems = [systems]
        if kind not in ("projection", "smoothness"):
            raise UsageError(f"unknown objective kind {kind!r}")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        sds = [system_data(s, kind, cfg.rho) for s in systems]
        sd0 = sds[0]
        for sd in sds[1:]:
            if sd.shape_key != sd0.shape_key or not (np.array_equal(sd.W, sd0.W)
                                                    and np.array_equal(sd.E, sd0.E)):
                raise ShapeError("all instances of a batch must share shape, basis and boundary rows")
        self.sd = sd0
        self.plan = get_plan(sd0, kind, cfg.rho, self.device.index)
        self.kind, self.cfg = kind, cfg
        n, n_d, n_xi = sd0.n, sd0.n_d, sd0.n_basis
        f64, dev = torch.float64, self.device
        h2d = [0]
        self.xi0 = _as_tensor(xi0, dev, f64, h2d)
        B = self.xi0.shape[0]
        if tuple(self.xi0.shape) != (B, n_d, n, n_xi):
            raise ShapeError(f"xi0 has shape {tuple(self.xi0.shape)}, expected (B, {n_d}, {n}, {n_xi})")
        self.B = B
        self.lam0 = (torch.zeros_like(self.xi0) if lam0 is None else _as_tensor(lam0, dev, f64, h2d))
        if tuple(self.lam0.shape) != tuple(self.xi0.shape):
            raise ShapeError("lam0 shape differs from xi0")
        if kind == "projection":
            if target is None:
                raise ShapeError("projection mode needs a target")
            self.target = _as_tensor(target, dev, f64, h2d)
            if tuple(self.target.shape) != tuple(self.xi0.shape):
                raise ShapeError("target shape differs from xi0")
        else:
            self.target = None
        if member_instance is None:
            if len(sds) != 1 and len(sds) != B:
                raise ShapeError("member_instance is required when instances != members")
            member_instance = np.zeros(B, np.int32) if len(sds) == 1 else np.arange(B, dtype=np.int32)
        mi = np.asarray(member_instance, np.int32)
        if mi.shape != (B,) or mi.min(initial=0) < 0 or mi.max(initial=0) >= len(sds):
            raise ShapeError("member_instance out of range")
        self.member_instance = _as_tensor(mi, dev, torch.int32, h2d)
        self.bvals = _as_tensor(np.stack([s.bvals for s in sds]), dev, f64, h2d)
        self.box = _as_tensor(np.stack([s.box for s in sds]), dev, f64, h2d)
        obs_np = np.stack([s.obs_pos for s in sds])
        self.obs_static = bool(obs_np.size == 0 or np.all(obs_np == obs_np[..., :1]))
        self.obs_pos = _as_tensor(obs_np, dev, f64, h2d)
        self.obs_axes = _as_tensor(np.stack([s.obs_axes for s in sds]), dev, f64, h2d)
        self.pair_axes = _as_tensor(np.stack([s.pair_axes for s in sds]), dev, f64, h2d)
        self.h2d_bytes = h2d[0]
        self.n_instances = len(sds)
        d_max = {s.d_max for s in sds}
        if len(d_max) != 1:
            raise ShapeError("all instances of a batch must share d_max")
        self.d_max = d_max.pop()
        self.early_exit = bool(early_exit)
        self.cluster = int(cluster)
        T = cfg.max_iters + 1
        self.out_xi = torch.empty_like(self.xi0)
        self.out_lam = torch.empty_like(self.xi0)
        self.out_primal = torch.empty(B, dtype=f64, device=dev)
        self.out_eq = torch.empty(B, dtype=f64, device=dev)
        self.out_its = torch.empty(B, dtype=torch.int32, device=dev)
        self.out_status = torch.empty(B, dtype=torch.int32, device=dev)
        self.out_trace = torch.empty((B, T, 2), dtype=f64, device=dev) if trace else None
        self.out_counters = torch.zeros((B, 4), dtype=torch.int64, device=dev) if counters else None
        self._build_structs()

    def _build_structs(self):
        p = lambda t: None if t is None else t.data_ptr()
        self._batch = _lib.Batch(self.B, self.n_instances, p(self.member_instance), p(self.xi0),
                                 p(self.lam0), p(self.target), p(self.bvals), p(self.box),
                                 p(self.obs_pos), p(self.obs_axes), p(self.pair_axes),
                                 _lib.BATCH_STATIC_OBSTACLES if self.obs_static else 0)
        c = self.cfg
        self._cfg = _lib.Config(float(c.rho), float(c.primal_tol), float(c.fp_tol),
                                float(self.d_max), int(c.max_iters), 1 if self.early_exit else 0,
                                self.cluster)
        self._out = _lib.Out(p(self.out_xi), p(self.out_lam), p(self.out_primal), p(self.out_eq),
                             p(self.out_its), p(self.out_status), p(self.out_trace),
                             p(self.out_counters))

    def launch(self, stream=None) -> None:
        """Enqueue the solve on `stream` (torch stream or None = current); no host sync."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _lib.lib().sfb_solve(self.plan.handle, ctypes.byref(self._batch), ctypes.byref(self._cfg),
                                  ctypes.byref(self._out), ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "sfb_solve")

    def results(self) -> dict:
        """Copy results to the host (synchronizes). Member-major arrays."""
        its = self.out_its.cpu().numpy()
        d2h = its.nbytes + sum(t.numel() * t.element_size() for t in
                               (self.out_xi, self.out_lam, self.out_primal, self.out_eq, self.out_status))
        out = {
            "xi": self.out_xi.cpu().numpy(), "lam": self.out_lam.cpu().numpy(),
            "primal": self.out_primal.cpu().numpy(), "eq_max": self.out_eq.cpu().numpy(),
            "iterations": its, "status": [_lib.STATUS[int(s)] for s in self.out_status.cpu().numpy()],
        }
        if self.out_trace is not None:
            T = int(its.max()) + 1 if its.size else 0
            tr = self.out_trace[:, :T].cpu().numpy()
            d2h += tr.nbytes
            out["trace"] = [tr[b, : its[b] + 1] for b in range(self.B)]
        if self.out_counters is not None:
            out["counters"] = self.out_counters.cpu().numpy()
        out["d2h_bytes"] = d2h
        return out


# ------------------------------------------------------------- reference API


def _target(mode, B: int):
    """solver.py:198-208 (broadcast and batch check), reference layout (n_d, nv, B)."""
    if mode.kind != "projection":
        return None
    t = np.asarray(mode.target, float)
    if t.ndim == 2:
        t = t[:, :, None]
    if t.shape[-1] == 1 and B > 1:
        t = np.broadcast_to(t, t.shape[:2] + (B,))
    if t.shape[-1] != B:
        raise ShapeError(f"projection target batch {t.shape[-1]} != state batch {B}")
    return t


def to_member_major(x: np.ndarray, n: int, n_xi: int) -> np.ndarray:
    """(n_d, n*n_xi, B) -> (B, n_d, n, n_xi)."""
    x = np.asarray(x, float)
    n_d, _, B = x.shape
    return np.ascontiguousarray(np.moveaxis(x, -1, 0).reshape(B, n_d, n, n_xi))


def solve_batch(init: SolverState, sys, mode: ObjectiveMode, cfg: SolverConfig | None = None,
                cache: KktCache | None = None) -> list[SolverResult]:
    """solver.py:286-355: run every member to its own convergence, on the GPU."""
    cfg = cfg or SolverConfig()
    kind = getattr(mode, "kind", None)
    if kind not in ("projection", "smoothness"):
        raise UsageError(f"unknown objective kind {kind!r}")
    if not isinstance(cache, KktCache) or cache.kind != kind or cache.rho != float(cfg.rho):
        cache = KktCache(sys, mode, cfg)
    t0 = time.perf_counter()
    B = init.xi.shape[-1]
    d = sys.dims
    tgt = _target(mode, B)
    xi0 = to_member_major(init.xi, d.n, d.n_basis)
    lam0 = to_member_major(init.lam, d.n, d.n_basis)
    t_mm = None if tgt is None else to_member_major(tgt, d.n, d.n_basis)
    batch = DeviceBatch([sys], xi0, lam0, t_mm, kind=kind, cfg=cfg, early_exit=True, trace=True)
    batch.launch()
    out = batch.results()
    wall = time.perf_counter() - t0
    res = []
    for b in range(B):
        res.append(SolverResult(
            xi=out["xi"][b].reshape(d.n_d, d.nvar_ax), lam=out["lam"][b].reshape(d.n_d, d.nvar_ax),
            status=out["status"][b], iterations=int(out["iterations"][b]),
            primal=float(out["primal"][b]), trace=out["trace"][b],
            eq_violation_max=float(out["eq_max"][b]), wall_time=wall))
    return res


def solve(init: SolverState, sys, mode: ObjectiveMode, cfg: SolverConfig | None = None,
          cache: KktCache | None = None) -> SolverResult:
    """solver.py:358-367."""
    if init.batch_size != 1:
        raise UsageError("solve expects a single-member state; use solve_batch")
    return solve_batch(init, sys, mode, cfg, cache)[0]


def fixed_point_step(state: SolverState, sys, mode: ObjectiveMode, cfg: SolverConfig,
                     cache: KktCache | None = None) -> SolverState:
    """solver.py:246-256: one map application (run as a 1-iteration fixed solve)."""
    B = state.batch_size
    d = sys.dims
    kind = getattr(mode, "kind", None)
    if kind not in ("projection", "smoothness"):
        raise UsageError(f"unknown objective kind {kind!r}")
    tgt = _target(mode, B)
    one = SolverConfig(rho=cfg.rho, max_iters=1, primal_tol=cfg.primal_tol, fp_tol=cfg.fp_tol,
                       d_max=cfg.d_max)
    batch = DeviceBatch([sys], to_member_major(state.xi, d.n, d.n_basis),
                        to_member_major(state.lam, d.n, d.n_basis),
                        None if tgt is None else to_member_major(tgt, d.n, d.n_basis),
                        kind=kind, cfg=one, early_exit=False, trace=False)
    batch.launch()
    out = batch.results()
    xi = np.moveaxis(out["xi"].reshape(B, d.n_d, d.nvar_ax), 0, -1)
    lam = np.moveaxis(out["lam"].reshape(B, d.n_d, d.nvar_ax), 0, -1)
    return SolverState(xi=xi, lam=lam, iteration=state.iteration + 1)


@dataclass
class BatchResult:
    xi: np.ndarray           # (B, n_d, n, n_basis)
    lam: np.ndarray
    status: list
    iterations: np.ndarray
    primal: np.ndarray
    eq_violation_max: np.ndarray
    trace: list | None = None
    counters: np.ndarray | None = None
    wall_time: float = 0.0
    extra: dict = field(default_factory=dict)


def solve_instances(systems, xi0, lam0=None, target=None, kind: str = "projection",
                    cfg: SolverConfig | None = None, member_instance=None,
                    fixed_iterations: bool = False, trace: bool = True,
                    cluster: int = 0) -> BatchResult:
    """Solve instances x samples in one launch (host arrays in, host arrays out).

    xi0/lam0/target: (B, n_d, n, n_basis) (numpy or torch, host or device);
    `systems[member_instance[b]]` is member b's constraint system. With
    fixed_iterations=True every member runs exactly cfg.max_iters + 1 map
    evaluations (the throughput protocol of SURVEY.md §8(d)). `cluster` = CTAs per
    member (0: auto — batches too small to fill the GPU split each member over a
    thread-block cluster for latency)."""
    cfg = cfg or SolverConfig()
    t0 = time.perf_counter()
    batch = DeviceBatch(systems, xi0, lam0, target, kind=kind, cfg=cfg,
                        member_instance=member_instance, early_exit=not fixed_iterations,
                        trace=trace, cluster=cluster)
    batch.launch()
    out = batch.results()
    return BatchResult(xi=out["xi"], lam=out["lam"], status=out["status"],
                       iterations=out["iterations"], primal=out["primal"],
                       eq_violation_max=out["eq_max"], trace=out.get("trace"),
                       wall_time=time.perf_counter() - t0,
                       extra={"h2d_bytes": batch.h2d_bytes, "d2h_bytes": out["d2h_bytes"]})


def cold_start(scn, sys) -> SolverState:
    """solver.py:144-148."""
    from .problem import straight_line_coeffs, xi_from_coeffs
    xi = xi_from_coeffs(straight_line_coeffs(scn.starts, scn.goals, sys.dims.n_basis))
    return SolverState(xi=xi, lam=np.zeros_like(xi))


def state_from_xi(xi: np.ndarray, lam: np.ndarray | None = None) -> SolverState:
    """solver.py:151-155."""
    if xi.ndim == 2:
        xi = xi[:, :, None]
    lam = np.zeros_like(xi) if lam is None else (lam[:, :, None] if lam.ndim == 2 else lam)
    return SolverState(xi=xi.astype(float), lam=lam.astype(float))
