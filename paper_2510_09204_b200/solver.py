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
class SphericalVars:
    """constraints.py:70-81: spherical reformulation variables, trailing batch axis.
    alpha/beta/d: (n_pairs, K+1, B); alpha_o/beta_o/d_o: (n, n_obs, K+1, B)."""

    alpha: np.ndarray
    beta: np.ndarray
    d: np.ndarray
    alpha_o: np.ndarray
    beta_o: np.ndarray
    d_o: np.ndarray


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


def _kron_checked(A: np.ndarray, n: int, E: np.ndarray) -> bool:
    """A == I_n (x) E: every diagonal block equals E and nothing outside the diagonal blocks
    is non-zero (a view and two reductions; no n x n Kronecker product is formed)."""
    nb, nx = E.shape
    if A.shape != (n * nb, n * nx):
        return False
    r = np.arange(n)
    diag = A.reshape(n, nb, n, nx)[r, :, r, :]           # (n, nb, nx)
    return bool(np.array_equal(diag, np.broadcast_to(E, diag.shape))
                and np.count_nonzero(A) == np.count_nonzero(diag))


_SD: dict = {}


def system_data(sys, kind: str = "projection", rho: float = 1.0) -> SystemData:
    """Extract and validate the structured data of a (reference or local) ConstraintSystem.

    Memoised per system object (weak reference + identities of its arrays): like the reference's
    KktCache (solver.py:64-91), a ConstraintSystem is treated as immutable once built."""
    import weakref
    arrs = (sys.A, sys.b, sys.h, sys.obs_pos, sys.obs_axes, sys.pair_axes, sys.basis.W)
    ident = tuple(map(id, arrs))
    hit = _SD.get(id(sys))
    if hit is not None and hit[0]() is sys and hit[1] == ident and hit[2] == float(sys.d_max):
        return hit[3]
    sd = _system_data(sys, kind, rho)
    if len(_SD) > 4096:
        _SD.clear()
    try:
        _SD[id(sys)] = (weakref.ref(sys), ident, float(sys.d_max), sd)
    except TypeError:                     # object without weakref support: no memo
        pass
    return sd


def _check_selection_structure(sys, W: np.ndarray) -> None:
    """The plan's KKT blocks assume the F, G and pair list `assemble` builds
    (constraints.py:122-139): every pair i < j in lexicographic order, then every
    (robot, obstacle) row, F = [D (x) W; I (x) (1_m (x) W)] and G = [I (x) W; -I (x) W].
    A reference system carrying its dense F / G is checked structurally (shapes, index
    lists, a fixed sample of rows) so a different selection is refused instead of being
    solved with the wrong KKT matrix."""
    d = sys.dims
    n, K1, n_xi, m = d.n, d.num_steps, d.n_basis, d.n_obs
    pairs = getattr(sys, "pair_index", None)
    if pairs is not None and [tuple(p) for p in pairs] != [(i, j) for i in range(n) for j in range(i + 1, n)]:
        raise UsageError("pair_index is not the full lexicographic pair list: unsupported constraint system")
    obs_index = getattr(sys, "obs_index", None)
    if obs_index is not None and [tuple(p) for p in obs_index] != [(i, o) for i in range(n) for o in range(m)]:
        raise UsageError("obs_index is not the full (robot, obstacle) list: unsupported constraint system")
    P = n * (n - 1) // 2
    F = getattr(sys, "F", None)
    if F is not None:
        F = np.asarray(F)
        if F.shape != ((P + n * m) * K1, n * n_xi):
            raise UsageError(f"F has shape {F.shape}, expected {((P + n * m) * K1, n * n_xi)}")
        rows = sorted({0, K1 - 1, P * K1 - 1, P * K1, F.shape[0] - 1, (P // 2) * K1 + K1 // 2}
                      & set(range(F.shape[0])))
        for r in rows:
            want = np.zeros(n * n_xi)
            k = r % K1
            if r < P * K1:
                i, j = [(i, j) for i in range(n) for j in range(i + 1, n)][r // K1]
                want[i * n_xi:(i + 1) * n_xi] = W[k]
                want[j * n_xi:(j + 1) * n_xi] = -W[k]
            else:
                i = (r - P * K1) // (m * K1)
                want[i * n_xi:(i + 1) * n_xi] = W[k]
            if not np.array_equal(F[r], want):
                raise UsageError(f"F row {r} is not the pair/obstacle selection of assemble: "
                                 "unsupported constraint system")
    G = getattr(sys, "G", None)
    if G is not None:
        G = np.asarray(G)
        if G.shape != (2 * n * K1, n * n_xi):
            raise UsageError(f"G has shape {G.shape}, expected {(2 * n * K1, n * n_xi)}")
        for r in sorted({0, K1 - 1, n * K1 - 1, n * K1, 2 * n * K1 - 1}):
            want = np.zeros(n * n_xi)
            i, k = (r % (n * K1)) // K1, r % K1
            want[i * n_xi:(i + 1) * n_xi] = W[k] if r < n * K1 else -W[k]
            if not np.array_equal(G[r], want):
                raise UsageError(f"G row {r} is not the workspace box of assemble: "
                                 "unsupported constraint system")


def _system_data(sys, kind: str, rho: float) -> SystemData:
    d = sys.dims
    n, n_d, n_xi, K1, m = d.n, d.n_d, d.n_basis, d.num_steps, d.n_obs
    A = np.asarray(sys.A, float)
    if A.shape[1] != n * n_xi or A.shape[0] % n != 0:
        if _dense_kkt_cond(sys, kind, rho) > 1e14:
            raise SetupError("KKT matrix is singular or near-singular")
        raise UsageError("boundary matrix A is not I_n (x) E: unsupported constraint system")
    nb = A.shape[0] // n
    E = A[:nb, :n_xi].copy()
    if not _kron_checked(A, n, E):
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
    _check_selection_structure(sys, W)
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


_PINNED: dict = {}


def _pinned(n: int, which: str = "in"):
    """Grow-only pinned host staging buffers (float64): the input arena ("in") and the
    output copies ("out", "trace"). Each use is synchronous, so reuse is safe."""
    import torch
    buf = _PINNED.get(which)
    if buf is None or buf.numel() < n:
        size = max(n, 1 << 16)
        try:
            buf = torch.empty(size, dtype=torch.float64).pin_memory()
        except RuntimeError:                      # no CUDA context yet / no pinning available
            buf = torch.empty(size, dtype=torch.float64)
        _PINNED[which] = buf
    return buf


SMALL_D2H_BYTES = 1 << 20   # output arenas up to this size are read back in one copy

_STREAM_SLOTS: list = []     # idle solve_stream slots (pinned in/out arenas), grow-only pool


def _checkout_slots(depth: int) -> list:
    """Take `depth` slots from the pool (new ones are empty and pin their arenas on first
    use). Pinning (cudaHostAlloc) costs 10-100+ ms and varies with host load, so a serving
    loop must not pay it per stream; slots go back to the pool when the stream ends."""
    got = []
    while _STREAM_SLOTS and len(got) < depth:
        got.append(_STREAM_SLOTS.pop())
    while len(got) < depth:
        got.append(dict(staging={}, out=None))
    for s in got:
        s["done"] = None
    return got


class DeviceBatch:
    """A batch of members (instance x sample) resident on one GPU.

    Inputs are member-major: xi0/lam0/target (B, n_d, n, n_basis). `systems` is one
    constraint system per instance (all with the same shape and basis);
    member_instance[b] selects member b's instance."""

    def __init__(self, systems, xi0, lam0=None, target=None, kind="projection", cfg=None,
                 member_instance=None, early_exit=True, trace=True, counters=False,
                 device=None, cluster=0, staging=None, copy_stream=None, layout="member"):
        """staging / copy_stream (solve_stream): a caller-owned pinned input arena and the
        stream the input copies are enqueued on (asynchronously); default: the shared
        staging buffer and synchronous copies.

        layout: "member" — xi0 / lam0 / target are (B, n_d, n, n_basis); "producer" — they
        are (B, n, n_d, n_basis), the layout of the reference's PyTorch producers (the flow
        sampler, flow_model.py:228-256, and InitNet.forward, init_net.py:74-96). A CUDA
        tensor in either layout and dtype (FP32 or FP64) is permuted / widened on the
        device, with no host round trip."""
        import torch
        cfg = cfg or SolverConfig()
        if not isinstance(systems, (list, tuple)):
            systems = [systems]
        if kind not in ("projection", "smoothness"):
            raise UsageError(f"unknown objective kind {kind!r}")
        if layout not in ("member", "producer"):
            raise UsageError(f"unknown coefficient layout {layout!r}")
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
        # ---- inputs: host arrays are packed into one buffer and cross PCIe in one copy;
        # CUDA tensors (e.g. straight from a PyTorch sampler) are used in place
        host_parts, dev_parts, uploaded = [], {}, {}
        direct_bytes = 0

        coeff_names = ("xi0", "lam0", "target")

        def add(name, x, shape, dtype=np.float64):
            nonlocal direct_bytes
            swap = layout == "producer" and name in coeff_names   # (B, n, n_d, c) -> (B, n_d, n, c)
            if swap:
                if x.ndim != 4:
                    raise ShapeError(f"{name} must be (B, n, n_d, n_basis), got {tuple(x.shape)}")
                if isinstance(x, torch.Tensor):
                    if x.shape[1:] != (n, n_d, n_xi):
                        raise ShapeError(f"{name} has shape {tuple(x.shape)}, expected (B, {n}, {n_d}, {n_xi})")
                    x = x.permute(0, 2, 1, 3)
                    if not x.is_cuda:
                        x = x.contiguous()
                else:
                    a = np.asarray(x)
                    if a.shape[1:] != (n, n_d, n_xi):
                        raise ShapeError(f"{name} has shape {a.shape}, expected (B, {n}, {n_d}, {n_xi})")
                    x = a.transpose(0, 2, 1, 3)
            if isinstance(x, torch.Tensor) and x.is_cuda:
                t = x.to(device=dev, dtype=torch.float64 if dtype == np.float64 else torch.int32)
                dev_parts[name] = t.contiguous()
                return tuple(t.shape)
            if (isinstance(x, torch.Tensor) and dtype == np.float64 and x.dtype == torch.float64
                    and x.is_contiguous() and x.is_pinned()):
                # pinned host tensor: one DMA straight from it (the same tensor passed as
                # xi0 and target crosses once)
                key = (x.data_ptr(), tuple(x.shape))
                if key not in uploaded:
                    if copy_stream is not None:
                        with torch.cuda.stream(copy_stream):
                            uploaded[key] = x.to(dev, non_blocking=True)
                    else:
                        uploaded[key] = x.to(dev)
                    direct_bytes += x.numel() * 8
                dev_parts[name] = uploaded[key]
                return tuple(x.shape)
            a = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x
            a = np.ascontiguousarray(np.asarray(a, dtype=dtype))
            host_parts.append((name, a))
            return a.shape

        xshape = add("xi0", xi0, None)
        B = xshape[0]
        if tuple(xshape) != (B, n_d, n, n_xi):
            raise ShapeError(f"xi0 has shape {tuple(xshape)}, expected (B, {n_d}, {n}, {n_xi})")
        self.B = B
        if lam0 is not None and add("lam0", lam0, None) != xshape:
            raise ShapeError("lam0 shape differs from xi0")
        if kind == "projection":
            if target is None:
                raise ShapeError("projection mode needs a target")
            if add("target", target, None) != xshape:
                raise ShapeError("target shape differs from xi0")
        if member_instance is None:
            if len(sds) != 1 and len(sds) != B:
                raise ShapeError("member_instance is required when instances != members")
            member_instance = np.zeros(B, np.int32) if len(sds) == 1 else np.arange(B, dtype=np.int32)
        mi = np.asarray(member_instance, np.int32)
        if mi.shape != (B,) or mi.min(initial=0) < 0 or mi.max(initial=0) >= len(sds):
            raise ShapeError("member_instance out of range")
        add("bvals", np.stack([q.bvals for q in sds]), None)
        add("box", np.stack([q.box for q in sds]), None)
        obs_np = np.stack([q.obs_pos for q in sds])
        self.obs_static = bool(obs_np.size == 0 or np.all(obs_np == obs_np[..., :1]))
        add("obs_pos", obs_np, None)
        add("obs_axes", np.stack([q.obs_axes for q in sds]), None)
        add("pair_axes", np.stack([q.pair_axes for q in sds]), None)
        # member_instance rides in the float64 arena as raw int32 words
        mi_words = np.zeros((B + 1) // 2 * 2, np.int32)
        mi_words[:B] = mi
        host_parts.append(("member_instance", mi_words.view(np.float64)))
        offs, total = {}, 0
        for name, a in host_parts:
            offs[name] = (total, a.shape)
            total += a.size
        if staging is None:
            staging = _pinned(total)
        else:                                      # caller-owned holder {"buf": pinned tensor}
            if staging.get("buf") is None or staging["buf"].numel() < total:
                staging["buf"] = torch.empty(max(total, 1 << 16), dtype=torch.float64).pin_memory()
            staging = staging["buf"]
        arena_h = staging.numpy()[:total]
        for name, a in host_parts:
            o, _ = offs[name]
            arena_h[o: o + a.size] = a.reshape(-1)
        if copy_stream is not None:
            with torch.cuda.stream(copy_stream):
                self._in_arena = staging[:total].to(dev, non_blocking=True)
        else:
            self._in_arena = staging[:total].to(dev)   # synchronous copy from pinned memory
        self.in_total = total
        self.h2d_bytes = int(arena_h.nbytes) + direct_bytes
        views = {}
        for name, (o, shp) in offs.items():
            views[name] = self._in_arena[o: o + int(np.prod(shp))].view(shp)
        views.update(dev_parts)
        self.xi0 = views["xi0"]
        self.lam0 = views.get("lam0")
        if self.lam0 is None:
            self.lam0 = torch.zeros_like(self.xi0)
        self.target = views.get("target") if kind == "projection" else None
        self.member_instance = views["member_instance"].view(torch.int32)[:B]
        self.bvals, self.box = views["bvals"], views["box"]
        self.obs_pos, self.obs_axes, self.pair_axes = views["obs_pos"], views["obs_axes"], views["pair_axes"]
        self.n_instances = len(sds)
        d_max = {q.d_max for q in sds}
        if len(d_max) != 1:
            raise ShapeError("all instances of a batch must share d_max")
        self.d_max = d_max.pop()
        self.early_exit = bool(early_exit)
        self.cluster = int(cluster)
        # ---- outputs: one arena, one device-to-host copy
        T = cfg.max_iters + 1
        nvm = B * n_d * n * n_xi
        seg = [("xi", nvm), ("lam", nvm), ("primal", B), ("eq", B), ("its", (B + 1) // 2),
               ("status", (B + 1) // 2)]
        if trace:
            seg.append(("trace", B * T * 2))
        oofs, ototal = {}, 0
        for name, sz in seg:
            oofs[name] = (ototal, sz)
            ototal += sz
        self._out_arena = torch.empty(ototal, dtype=f64, device=dev)
        ov = {k: self._out_arena[o: o + sz] for k, (o, sz) in oofs.items()}
        self.out_xi = ov["xi"].view(B, n_d, n, n_xi)
        self.out_lam = ov["lam"].view(B, n_d, n, n_xi)
        self.out_primal, self.out_eq = ov["primal"], ov["eq"]
        self.out_its = ov["its"].view(torch.int32)[:B]
        self.out_status = ov["status"].view(torch.int32)[:B]
        self.out_trace = ov["trace"].view(B, T, 2) if trace else None
        self._out_prefix = oofs["status"][0] + oofs["status"][1]   # everything but the trace
        self._oofs = oofs
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

    def analysis(self, which: str = "xi0"):
        """The reference's _analyze intermediates (solver.py:158-169) of the batch's input
        coefficients (which="xi0") or of the solved ones ("xi"), computed on the GPU by
        sfb_analysis_vars: (SphericalVars, s) in the reference's layouts (batch axis last);
        s = max(0, h - G xi) is (n_d, 2 n K1, B)."""
        import torch
        sd, B = self.sd, self.B
        n, n_d, K1, m = sd.n, sd.n_d, sd.num_steps, sd.n_obs
        P = n * (n - 1) // 2
        dev, f64 = self.device, torch.float64
        x = (self.xi0 if which == "xi0" else self.out_xi).contiguous()
        self._wait_launch()
        Wd = torch.from_numpy(np.ascontiguousarray(sd.W)).to(dev)
        alpha, beta, dd = (torch.empty((P, K1, B), dtype=f64, device=dev) for _ in range(3))
        alpha_o, beta_o, d_o = (torch.empty((n, m, K1, B), dtype=f64, device=dev) for _ in range(3))
        slack = torch.empty((n_d, 2 * n * K1, B), dtype=f64, device=dev)
        p = lambda t: t.data_ptr() if t.numel() else None
        stream = torch.cuda.current_stream(dev)
        rc = _lib.lib().sfb_analysis_vars(
            x.data_ptr(), B, self.member_instance.data_ptr(), n_d, n, sd.n_basis, K1, m, Wd.data_ptr(),
            self.pair_axes.data_ptr(), p(self.obs_axes), p(self.obs_pos), self.box.data_ptr(),
            float(self.d_max), p(alpha), p(beta), p(dd), p(alpha_o), p(beta_o), p(d_o),
            slack.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
        _lib.check(rc, "sfb_analysis_vars")
        h = lambda t: t.cpu().numpy()
        return SphericalVars(h(alpha), h(beta), h(dd), h(alpha_o), h(beta_o), h(d_o)), h(slack)

    def launch_info(self) -> dict:
        """Cluster size, shared memory per CTA and resident CTAs per SM of this batch's launch."""
        c, sm, k = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        flags = _lib.BATCH_STATIC_OBSTACLES if self.obs_static else 0
        rc = _lib.lib().sfb_launch_info(self.plan.handle, int(self.B), int(self.cluster), flags,
                                        ctypes.byref(c), ctypes.byref(sm), ctypes.byref(k))
        _lib.check(rc, "sfb_launch_info")
        return {"cluster": c.value, "smem_bytes": sm.value, "ctas_per_sm": k.value}

    def launch(self, stream=None) -> None:
        """Enqueue the solve on `stream` (torch stream or None = current); no host sync."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _lib.lib().sfb_solve(self.plan.handle, ctypes.byref(self._batch), ctypes.byref(self._cfg),
                                  ctypes.byref(self._out), ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "sfb_solve")
        # results() copies on the current stream: it waits for this event, so a launch on
        # any other stream is complete before its outputs are read
        self._done = torch.cuda.Event()
        self._done.record(s)

    def _wait_launch(self):
        import torch
        ev = getattr(self, "_done", None)
        if ev is not None:
            torch.cuda.current_stream(self.device).wait_event(ev)

    def results(self) -> dict:
        """Copy results to the host (synchronizes): one copy of the output arena (the trace
        only up to the longest member's iterations). Member-major arrays."""
        B, n_d, n, n_xi = self.out_xi.shape
        self._wait_launch()
        # a small arena (the latency case) crosses in one copy with the whole trace; a large
        # one copies the head first, then the trace only up to the longest member's iterations
        one_copy = self.out_trace is not None and self._out_arena.numel() * 8 <= SMALL_D2H_BYTES
        nh = self._out_arena.numel() if one_copy else self._out_prefix
        head = _pinned(nh, "out")[:nh]
        head.copy_(self._out_arena[:nh])
        head = head.numpy()
        o = self._oofs
        get = lambda k: head[o[k][0]: o[k][0] + o[k][1]]
        its = get("its").view(np.int32)[:B].copy()
        st = get("status").view(np.int32)[:B]
        out = {
            "xi": get("xi").reshape(B, n_d, n, n_xi).copy(), "lam": get("lam").reshape(B, n_d, n, n_xi).copy(),
            "primal": get("primal").copy(), "eq_max": get("eq").copy(),
            "iterations": its, "status": [_lib.STATUS[int(v)] for v in st],
        }
        d2h = head.nbytes
        if self.out_trace is not None:
            T = int(its.max()) + 1 if its.size else 0
            if one_copy:
                tr = get("trace").reshape(B, -1, 2)[:, :T].copy()
            else:
                tr = _pinned(B * T * 2, "trace")[: B * T * 2].view(B, T, 2)
                tr.copy_(self.out_trace[:, :T])
                tr = tr.numpy().copy()
                d2h += tr.nbytes
            out["trace"] = [tr[b, : its[b] + 1] for b in range(B)]
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
    """solver.py:246-256: one map application (run as a 1-iteration fixed solve). Like the
    reference, the returned state carries the slack `s` (n_d, g_rows, B) and the spherical
    variables `vars` of the INPUT iterate (computed on the GPU, sfb_analysis_vars)."""
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
    vars_, s = batch.analysis("xi0")
    xi = np.moveaxis(out["xi"].reshape(B, d.n_d, d.nvar_ax), 0, -1)
    lam = np.moveaxis(out["lam"].reshape(B, d.n_d, d.nvar_ax), 0, -1)
    return SolverState(xi=xi, lam=lam, s=s, vars=vars_, iteration=state.iteration + 1)


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
                    cluster: int = 0, layout: str = "member") -> BatchResult:
    """Solve instances x samples in one launch (host arrays in, host arrays out).

    xi0/lam0/target: (B, n_d, n, n_basis) (numpy or torch, host or device);
    `systems[member_instance[b]]` is member b's constraint system. With
    fixed_iterations=True every member runs exactly cfg.max_iters + 1 map
    evaluations (the throughput protocol of SURVEY.md §8(d)). `cluster` = CTAs per
    member (0: auto — batches too small to fill the GPU split each member over a
    thread-block cluster for latency). layout="producer": the coefficients are
    (B, n, n_d, n_basis) as the reference's sampler / init network emit them (see
    DeviceBatch); results are member-major either way."""
    cfg = cfg or SolverConfig()
    t0 = time.perf_counter()
    batch = DeviceBatch(systems, xi0, lam0, target, kind=kind, cfg=cfg,
                        member_instance=member_instance, early_exit=not fixed_iterations,
                        trace=trace, cluster=cluster, layout=layout)
    batch.launch()
    out = batch.results()
    return BatchResult(xi=out["xi"], lam=out["lam"], status=out["status"],
                       iterations=out["iterations"], primal=out["primal"],
                       eq_violation_max=out["eq_max"], trace=out.get("trace"),
                       wall_time=time.perf_counter() - t0,
                       extra={"h2d_bytes": batch.h2d_bytes, "d2h_bytes": out["d2h_bytes"]})


def solve_stream(steps, kind: str = "projection", cfg: SolverConfig | None = None,
                 fixed_iterations: bool = False, trace: bool = True, cluster: int = 0, depth: int = 3):
    """Pipelined solve_instances over a sequence of batches (the serving loop): yields one
    BatchResult per step, in order. `steps` yields (systems, xi0, lam0, target,
    member_instance) tuples of host (or CUDA) arrays.

    Every step still packs its inputs into a pinned arena, copies them to the device and
    reads its whole output arena back; those copies run on a copy stream and the host
    packing runs ahead, so they overlap the neighbouring steps' kernels. `depth` steps are in
    flight (pinned and device arenas per slot; step k + depth reuses step k's buffers only after
    step k's copies completed): the host may fall behind by depth - 1 kernels (scheduling
    jitter on a busy host) before the GPU idles."""
    depth = max(2, int(depth))
    import torch
    cfg = cfg or SolverConfig()
    dev = torch.device("cuda", torch.cuda.current_device())
    compute = torch.cuda.current_stream(dev)
    copy_in, copy_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)   # H2D of step k+1 must
    # not queue behind the D2H of step k (which waits for kernel k)
    slots = _checkout_slots(depth)
    pending = []    # (batch, slot, d2h event, t0)

    def finish(item):
        batch, slot, ev, t0 = item
        ev.synchronize()
        head = slot["out"].numpy()
        o = batch._oofs
        B, n_d, n, n_xi = batch.out_xi.shape
        get = lambda k: head[o[k][0]: o[k][0] + o[k][1]]
        its = get("its").view(np.int32)[:B].copy()
        st = get("status").view(np.int32)[:B]
        tr = None
        if batch.out_trace is not None:
            T = batch.out_trace.shape[1]
            full = get("trace").reshape(B, T, 2)
            tr = [full[b, : its[b] + 1].copy() for b in range(B)]
        return BatchResult(xi=get("xi").reshape(B, n_d, n, n_xi).copy(),
                           lam=get("lam").reshape(B, n_d, n, n_xi).copy(),
                           status=[_lib.STATUS[int(v)] for v in st], iterations=its,
                           primal=get("primal").copy(), eq_violation_max=get("eq").copy(),
                           trace=tr, wall_time=time.perf_counter() - t0,
                           extra={"h2d_bytes": batch.h2d_bytes,
                                  "d2h_bytes": int(batch._out_arena.numel()) * 8})

    try:
        yield from _stream_loop(steps, slots, pending, finish, depth, compute, copy_in, copy_out,
                                kind, cfg, fixed_iterations, trace, cluster)
    finally:
        for s in slots:                           # copies still in flight finish before reuse
            if s["done"] is not None:
                s["done"].synchronize()
        _STREAM_SLOTS.extend(slots)


def _stream_loop(steps, slots, pending, finish, depth, compute, copy_in, copy_out,
                 kind, cfg, fixed_iterations, trace, cluster):
    import torch
    for k, (systems, xi0, lam0, target, mi) in enumerate(steps):
        t0 = time.perf_counter()
        slot = slots[k % depth]
        if slot["done"] is not None:
            slot["done"].synchronize()            # this slot's copies of step k - depth completed
        batch = DeviceBatch(systems, xi0, lam0, target, kind=kind, cfg=cfg, member_instance=mi,
                            early_exit=not fixed_iterations, trace=trace, cluster=cluster,
                            staging=slot["staging"], copy_stream=copy_in)
        batch._in_arena.record_stream(compute)
        ev_in = torch.cuda.Event()
        ev_in.record(copy_in)
        compute.wait_event(ev_in)
        batch.launch(compute)
        ev_k = torch.cuda.Event()
        ev_k.record(compute)
        nout = batch._out_arena.numel()
        if slot["out"] is None or slot["out"].numel() < nout:
            slot["out"] = torch.empty(nout, dtype=torch.float64).pin_memory()
        copy_out.wait_event(ev_k)
        with torch.cuda.stream(copy_out):
            slot["out"][:nout].copy_(batch._out_arena, non_blocking=True)
        batch._out_arena.record_stream(copy_out)
        ev_out = torch.cuda.Event()
        ev_out.record(copy_out)
        slot["done"] = ev_out
        pending.append((batch, dict(out=slot["out"][:nout]), ev_out, t0))
        if len(pending) >= depth:
            yield finish(pending.pop(0))
    while pending:
        yield finish(pending.pop(0))


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


# ------------------------------------------------ callers either side of the solve


def batch_primal_residual(xi, sys) -> np.ndarray:
    """solver.py:185-187: primal residual of every member of xi (n_d, nv, B), on the GPU
    (the map's analysis half only: a zero-iteration solve). The planner ranks its
    candidates by this value (pipeline.py:113-115)."""
    xi = np.asarray(xi, float)
    if xi.ndim == 2:
        xi = xi[:, :, None]
    d = sys.dims
    mm = to_member_major(xi, d.n, d.n_basis)
    cfg = SolverConfig(max_iters=0, d_max=float(sys.d_max))
    out = solve_instances([sys], mm, None, mm, cfg=cfg, fixed_iterations=True, trace=False)
    return np.asarray(out.primal, float)


def primal_residual(state: SolverState, sys):
    """solver.py:177-182."""
    out = batch_primal_residual(state.xi, sys)
    return float(out[0]) if out.size == 1 else out


def rank_candidates(xi_all, sys) -> tuple[np.ndarray, np.ndarray]:
    """Stage 1 of pipeline.plan (pipeline.py:113-115): residuals and the stable order."""
    pre = batch_primal_residual(xi_all, sys)
    return pre, np.argsort(pre, kind="stable")


def kinematic_peaks(xi_mm, basis, dense_factor: int = 10):
    """Largest speed / acceleration norm per member over robots and the dense grid of
    time_scale_for_limits (basis.py:134-139), computed on the GPU.
    xi_mm: (B, n_d, n, n_basis) member-major coefficients (numpy or CUDA tensor)."""
    import torch
    from .problem import BasisConfig, build_basis
    cfg = basis.config
    dense = build_basis(BasisConfig(cfg.n_basis, dense_factor * (cfg.num_steps - 1) + 1, cfg.duration))
    dev = torch.device("cuda", torch.cuda.current_device())
    x = xi_mm if isinstance(xi_mm, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(xi_mm, float))
    x = x.to(device=dev, dtype=torch.float64).contiguous()
    B, n_d, n, n_xi = x.shape
    wd = torch.from_numpy(np.ascontiguousarray(dense.Wd)).to(dev)
    wdd = torch.from_numpy(np.ascontiguousarray(dense.Wdd)).to(dev)
    out = torch.empty((2, B), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    rc = _lib.lib().sfb_kinematic_peaks(x.data_ptr(), B, n_d, n, n_xi, wd.data_ptr(), wdd.data_ptr(),
                                        dense.Wd.shape[0], out[0].data_ptr(), out[1].data_ptr(),
                                        ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc, "sfb_kinematic_peaks")
    o = out.cpu().numpy()
    return o[0], o[1]


def time_scale_batch(xi_mm, basis, v_max: float, a_max: float, dense_factor: int = 10) -> np.ndarray:
    """gamma = max(1, vhat/v_max, sqrt(ahat/a_max)) per member (basis.py:119-142)."""
    from .errors import ConfigError
    if not (v_max > 0 and a_max > 0):
        raise ConfigError("v_max and a_max must be positive")
    vhat, ahat = kinematic_peaks(xi_mm, basis, dense_factor)
    return np.maximum(1.0, np.maximum(vhat / v_max, np.sqrt(ahat / a_max)))


def time_scale_for_limits(coeffs, basis, v_max: float, a_max: float, dense_factor: int = 10):
    """basis.py:119-142 (single trajectory set (n, n_d, n_basis)): returns (gamma, basis
    rebuilt with duration gamma*T)."""
    from .problem import BasisConfig, build_basis
    c = np.asarray(coeffs, float)
    mm = c.transpose(1, 0, 2)[None]
    gamma = float(time_scale_batch(mm, basis, v_max, a_max, dense_factor)[0])
    cfg = basis.config
    return gamma, build_basis(BasisConfig(cfg.n_basis, cfg.num_steps, gamma * cfg.duration))
