"""ORACLE (test infrastructure only) — delta-form, Kronecker-KKT FP64 restatement.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import
this module; the product never does.

It computes the same map as the reference `_step` (pkg/src/swarmplan/solver.py:211-243)
through exact algebraic rewrites (derivations in DESIGN.md §3 and SURVEY.md App. A)
and is the algorithm the CUDA kernel implements, so the kernel is debugged against
it at sizes the dense oracle cannot reach (n = 64, 128):

1. trig-free projection: for a row with relative position delta and axes (a, b),
   rho = sqrt((dx^2 + dy^2)/a^2 + dz^2/b^2) equals the reference's num/den
   (constraints.py:166-192), and e = (clip(rho, 1, d_max)/rho) * delta
   (constraints.py:216-247), so r1 = delta * (1 - clip(rho, 1, d_max)/rho);
   coincident rows (rho = 0) use alpha = 0, beta = pi/2: r1 = (-a, 0, -b cos(pi/2)).
2. F^T r1 + G^T r2 = (I_n (x) W^T) g with g_i(k) = sum_{j>i} r1(i,j,k) - sum_{j<i} r1(j,i,k)
   + sum_o r1(i,o,k) + max(p - p_max, 0) - max(p_min - p, 0)  (F, G: constraints.py:122-137).
3. delta form of the KKT step (solver.py:231-241):
   xi+ = xi + Mxx (2 lam+ - lam + t - Q xi) + Mxb (b - A xi).
4. Kronecker inverse: H = I_n (x) Qb + rho((n+m+2) I - 11^T) (x) W^T W and A = I_n (x) E,
   so Mxx = I (x) Pxx + (1/n) 11^T (x) (Rxx - Pxx) (same for Mxb) with
   P = K(n+m+2)^-1, R = K(m+2)^-1, K(c) = [[Qb + rho c W^T W, E^T], [E, 0]].
   cond(M) = max|eig| / min|eig| over K(m+2) and (if n > 1) K(n+m+2).

Parity status: pinned — `tests/test_oracle.py` checks it against the reference
golden vectors (`tests/golden/*.npz`) and against `sf_dense` at ~1e-12.
"""

from __future__ import annotations

import numpy as np

COS_HALF_PI = float(np.cos(0.5 * np.pi))  # the reference's cos(beta) at beta = pi/2


def kkt_blocks(W, Wdd, E, n, m, kind, rho):
    """Return (Pxx, Pxb, Rxx, Rxb, cond) of the Kronecker-compressed KKT inverse."""
    n_xi = W.shape[1]
    nb = E.shape[0]
    S = W.T @ W
    Qb = np.eye(n_xi) if kind == "projection" else Wdd.T @ Wdd

    def K(c):
        k = np.zeros((n_xi + nb, n_xi + nb))
        k[:n_xi, :n_xi] = Qb + rho * c * S
        k[:n_xi, n_xi:] = E.T
        k[n_xi:, :n_xi] = E
        return k

    Km = K(m + 2)
    blocks = [Km]
    Kd = K(n + m + 2)
    if n > 1:
        blocks.append(Kd)
    ev = np.concatenate([np.abs(np.linalg.eigvalsh(b)) for b in blocks])
    cond = np.inf if ev.min() == 0 else ev.max() / ev.min()
    R = np.linalg.inv(Km)
    P = np.linalg.inv(Kd) if n > 1 else R
    return P[:n_xi, :n_xi], P[:n_xi, n_xi:], R[:n_xi, :n_xi], R[:n_xi, n_xi:], cond


def _r1(delta, a, b, d_max, n_d):
    """Trig-free residual of constraints.py:166-247 for rows delta (n_d, ...)."""
    q = (delta[0] ** 2 + delta[1] ** 2) / a**2
    if n_d == 3:
        q = q + delta[2] ** 2 / b**2
    rho = np.sqrt(q)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        f = np.where(rho < 1.0, 1.0 - 1.0 / rho,
                     np.where(rho > d_max, 1.0 - d_max / rho, 0.0))
    with np.errstate(invalid="ignore"):
        r1 = delta * f
    zero = rho == 0.0
    if np.any(zero):
        r1 = np.where(zero, 0.0, r1)
        r1[0] = np.where(zero, -a + 0.0 * delta[0], r1[0])
        if n_d == 3:
            r1[2] = np.where(zero, -b * COS_HALF_PI + 0.0 * delta[2], r1[2])
    return r1


class KronSF:
    """Per-system constants and the vectorized map over members."""

    def __init__(self, sys, kind: str, rho: float):
        d = sys.dims
        self.n, self.n_d, self.n_xi, self.K1, self.m = d.n, d.n_d, d.n_basis, d.num_steps, d.n_obs
        self.W = np.asarray(sys.basis.W, float)
        A = np.asarray(sys.A, float)
        self.nb = A.shape[0] // self.n
        self.E = A[: self.nb, : self.n_xi]
        self.b = np.asarray(sys.b, float).reshape(self.n_d, self.n, self.nb)
        h = np.asarray(sys.h, float)
        nk = self.n * self.K1
        self.pmax = h[:, :nk].reshape(self.n_d, self.n, self.K1)
        self.pmin = -h[:, nk:].reshape(self.n_d, self.n, self.K1)
        self.pair_axes = np.asarray(sys.pair_axes, float)
        self.obs_axes = np.asarray(sys.obs_axes, float)
        self.obs_pos = np.asarray(sys.obs_pos, float)  # (n_d, m, K1)
        self.d_max = float(sys.d_max)
        self.kind, self.rho = kind, float(rho)
        Wdd = np.asarray(sys.basis.Wdd, float)
        self.Qb = np.eye(self.n_xi) if kind == "projection" else Wdd.T @ Wdd
        self.Pxx, self.Pxb, self.Rxx, self.Rxb, self.cond = kkt_blocks(
            self.W, Wdd, self.E, self.n, self.m, kind, rho)

    def analyze(self, c):
        """c: (B, n_d, n, n_xi) -> g (B, n_d, n, n_xi) = F^T r1 + G^T r2, primal (B,), active rows."""
        n, n_d, m = self.n, self.n_d, self.m
        pos = np.einsum("kc,banc->bank", self.W, c)
        g = np.zeros_like(pos)
        s1 = np.zeros(c.shape[0])
        active = 0
        if n > 1:
            delta = pos[:, :, :, None, :] - pos[:, :, None, :, :]    # (B, n_d, i, j, K1)
            dl = np.moveaxis(delta, 1, 0)
            r1 = _r1(dl, self.pair_axes[0], self.pair_axes[2], self.d_max, n_d)
            iu = np.triu(np.ones((n, n), bool), 1)
            # owner i of row (i, j), i < j: +r1 ; owner j: -r1 (incl. the coincident rule)
            r1u = np.where(iu[None, None, :, :, None], r1, 0.0)
            g += np.moveaxis(r1u.sum(axis=3) - r1u.sum(axis=2), 0, 1)
            s1 += np.einsum("abijk,abijk->b", r1u, r1u)
            active += int(np.count_nonzero(np.any(r1u != 0.0, axis=0)))
        if m:
            dl = pos[:, :, :, None, :] - self.obs_pos[None, :, None, :, :]  # (B, n_d, i, o, K1)
            dl = np.moveaxis(dl, 1, 0)
            ao = self.obs_axes[:, 0][None, None, :, None]
            bo = self.obs_axes[:, 2][None, None, :, None]
            r1 = _r1(dl, ao, bo, self.d_max, n_d)
            g += np.moveaxis(r1.sum(axis=3), 0, 1)
            s1 += np.einsum("abiok,abiok->b", r1, r1)
            active += int(np.count_nonzero(np.any(r1 != 0.0, axis=0)))
        up = np.maximum(pos - self.pmax[None], 0.0)
        lo = np.maximum(self.pmin[None] - pos, 0.0)
        g += up - lo
        s2 = np.einsum("bank,bank->b", up, up) + np.einsum("bank,bank->b", lo, lo)
        G = np.einsum("kc,bank->banc", self.W, g)
        return G, np.sqrt(s1) + np.sqrt(s2), active

    def step(self, c, lam, t):
        """One map application in member-major layout (B, n_d, n, n_xi)."""
        G, primal, active = self.analyze(c)
        lam_new = lam - self.rho * G
        qc = c if self.kind == "projection" else np.einsum("cd,band->banc", self.Qb, c)
        delta = 2.0 * lam_new - lam + t - qc
        u = self.b[None] - np.einsum("rc,banc->banr", self.E, c)
        n = self.n
        c_new = (c + np.einsum("cd,band->banc", self.Pxx, delta)
                 + np.einsum("cr,banr->banc", self.Pxb, u)
                 + (np.einsum("cd,bad->bac", self.Rxx - self.Pxx, delta.sum(axis=2))
                    + np.einsum("cr,bar->bac", self.Rxb - self.Pxb, u.sum(axis=2)))[:, :, None, :] / n)
        return c_new, lam_new, primal, active

    def eq_violation(self, c):
        return np.abs(np.einsum("rc,banc->banr", self.E, c) - self.b[None]).max(axis=(1, 2, 3))


def to_member_major(x, n, n_xi):
    """(n_d, n*n_xi, B) reference layout -> (B, n_d, n, n_xi)."""
    n_d, _, B = x.shape
    return np.array(np.moveaxis(x, -1, 0).reshape(B, n_d, n, n_xi), dtype=float, copy=True)


def solve_batch(sys, xi0, lam0, kind="projection", target=None, rho=1.0, max_iters=15000,
                primal_tol=1e-3, fp_tol=1e-8, sf: KronSF | None = None, count_active=False,
                early_exit=True):
    """Same loop semantics as solver.py:286-355; inputs in the reference layout.

    early_exit=False runs exactly max_iters + 1 map evaluations (the fixed-iteration
    protocol): the reference's trig round-off keeps its primal > 1e-300, while this
    trig-free map can return an exact 0 for inactive rows."""
    early = bool(early_exit)
    sf = sf or KronSF(sys, kind, rho)
    n, n_xi = sf.n, sf.n_xi
    c = to_member_major(np.asarray(xi0, float), n, n_xi)
    lam = to_member_major(np.asarray(lam0, float), n, n_xi)
    B = c.shape[0]
    if kind == "projection":
        t = np.asarray(target, float)
        if t.ndim == 2:
            t = t[:, :, None]
        if t.shape[-1] == 1 and B > 1:
            t = np.broadcast_to(t, t.shape[:2] + (B,))
        t = to_member_major(t, n, n_xi)
    else:
        t = np.zeros_like(c)
    traces = [[] for _ in range(B)]
    status = ["max_iters"] * B
    eq_max = np.zeros(B)
    last_fp = np.full(B, np.inf)
    active = np.arange(B)
    rows_active = 0
    for it in range(max_iters + 1):
        cn, ln, primal, act = sf.step(c[active], lam[active], t[active])
        rows_active += act
        for p, b in enumerate(active):
            traces[b].append((float(primal[p]), float(last_fp[b])))
        conv_p = (primal < primal_tol) & (it >= 1) & early
        conv_f = (last_fp[active] < fp_tol) & early
        for p, b in enumerate(active):
            if conv_p[p]:
                status[b] = "converged_primal"
            elif conv_f[p]:
                status[b] = "converged_fp"
        keep = ~(conv_p | conv_f)
        if it == max_iters or not keep.any():
            break
        active = active[keep]
        cn, ln = cn[keep], ln[keep]
        last_fp[active] = ((cn - c[active]) ** 2).sum(axis=(1, 2, 3)) + \
            ((ln - lam[active]) ** 2).sum(axis=(1, 2, 3))
        c[active] = cn
        lam[active] = ln
        eq_max[active] = np.maximum(eq_max[active], sf.eq_violation(cn))
    tr = [np.array(x) for x in traces]
    out = {
        "xi": c.reshape(B, sf.n_d, n * n_xi), "lam": lam.reshape(B, sf.n_d, n * n_xi),
        "status": status, "iterations": np.array([len(x) - 1 for x in tr]),
        "primal": np.array([x[-1, 0] for x in tr]), "trace": tr, "eq_max": eq_max,
    }
    if count_active:
        out["active_rows"] = rows_active
    return out
