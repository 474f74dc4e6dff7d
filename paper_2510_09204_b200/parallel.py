"""Multi-GPU: instances shard across ranks (one process per GPU, torchrun); members
never interact, so the only collective is one NCCL gather of the final results to
the destination rank. No collective runs inside the iterations.
"""

from __future__ import annotations

import numpy as np

RESULT_FIELDS = ("xi", "lam", "primal", "eq_max", "iterations", "status")


def shard(n_instances: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous instance block [lo, hi) of `rank` (sizes differ by at most one)."""
    base, rem = divmod(n_instances, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def pack(fields: dict, B_pad: int, trace_len: int | None = None):
    """Flatten per-member results into one float64 tensor [B_pad, row] (padded rows = 0)."""
    import torch
    B = fields["xi"].shape[0]
    parts = [fields["xi"].reshape(B, -1), fields["lam"].reshape(B, -1),
             fields["primal"].reshape(B, 1), fields["eq_max"].reshape(B, 1),
             fields["iterations"].reshape(B, 1).to(torch.float64),
             fields["status"].reshape(B, 1).to(torch.float64),
             torch.ones(B, 1, dtype=torch.float64, device=fields["xi"].device)]  # valid flag
    if trace_len is not None:
        parts.append(fields["trace"][:, :trace_len].reshape(B, -1))
    flat = torch.cat([p.to(torch.float64) for p in parts], dim=1)
    if B_pad > B:
        flat = torch.cat([flat, flat.new_zeros(B_pad - B, flat.shape[1])])
    return flat.contiguous()


def unpack(flat, n_d: int, n: int, n_xi: int, trace_len: int | None = None) -> dict:
    """Inverse of `pack` on the host; drops padded rows."""
    a = flat.cpu().numpy()
    a = a[a[:, 2 * n_d * n * n_xi + 4] == 1.0]
    nv = n_d * n * n_xi
    out = {"xi": a[:, :nv].reshape(-1, n_d, n, n_xi), "lam": a[:, nv:2 * nv].reshape(-1, n_d, n, n_xi),
           "primal": a[:, 2 * nv], "eq_max": a[:, 2 * nv + 1],
           "iterations": a[:, 2 * nv + 2].astype(np.int64), "status": a[:, 2 * nv + 3].astype(np.int64)}
    if trace_len is not None:
        out["trace"] = a[:, 2 * nv + 5:].reshape(-1, trace_len, 2)
    return out


def gather_fields(fields: dict, B_pad: int, dst: int = 0, trace_len: int | None = None, group=None):
    """Gather every rank's packed results to `dst` (NCCL for CUDA tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    flat = pack(fields, B_pad, trace_len)
    if flat.is_cuda and dist.get_backend(group) == "gloo":   # gloo gathers host tensors only
        flat = flat.cpu()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [torch.empty_like(flat) for _ in range(world)] if rank == dst else None
    dist.gather(flat, bucket, dst=dst, group=group)
    return None if bucket is None else torch.cat(bucket)


def gather_results(batch, dst: int = 0, B_pad: int | None = None, trace: bool = False, group=None):
    """Gather a DeviceBatch's results (stream-ordered, no host sync on non-dst ranks)."""
    f = {"xi": batch.out_xi, "lam": batch.out_lam, "primal": batch.out_primal,
         "eq_max": batch.out_eq, "iterations": batch.out_its, "status": batch.out_status}
    T = None
    if trace and batch.out_trace is not None:
        f["trace"] = batch.out_trace
        T = batch.out_trace.shape[1]
    return gather_fields(f, B_pad or batch.B, dst, T, group)


def solve_sharded(systems, xi0, target=None, lam0=None, member_instance=None, kind="projection",
                  cfg=None, fixed_iterations=False, dst=0):
    """Each rank solves its contiguous block of instances; rank `dst` returns the full
    member-major results (dict), other ranks None. Inputs are the full (global) batch."""
    import torch.distributed as dist
    from .solver import DeviceBatch
    world, rank = dist.get_world_size(), dist.get_rank()
    I = len(systems)
    mi = np.zeros(xi0.shape[0], np.int64) if member_instance is None else np.asarray(member_instance)
    lo, hi = shard(I, world, rank)
    sel = np.flatnonzero((mi >= lo) & (mi < hi))
    counts = [int(np.count_nonzero((mi >= a) & (mi < b)))
              for a, b in (shard(I, world, r) for r in range(world))]
    B_pad = max(counts)
    take = lambda x: None if x is None else np.asarray(x)[sel]
    batch = DeviceBatch(systems[lo:hi], take(xi0), take(lam0), take(target), kind=kind, cfg=cfg,
                        member_instance=(mi[sel] - lo).astype(np.int32),
                        early_exit=not fixed_iterations, trace=False)
    batch.launch()
    flat = gather_results(batch, dst=dst, B_pad=B_pad)
    if flat is None:
        return None
    d = batch.sd
    return unpack(flat, d.n_d, d.n, d.n_basis)
