"""Multi-GPU: instances shard across ranks (one process per GPU, torchrun); members
never interact, so the only collective is one NCCL gather of the final results to
the destination rank. No collective runs inside the iterations.

Every gathered row carries its member's global index, so the destination rank
puts each result back at the member's position in the caller's batch whatever the
member -> instance map looks like (interleaved samples, ranks without instances).
"""

from __future__ import annotations

import numpy as np

RESULT_FIELDS = ("xi", "lam", "primal", "eq_max", "iterations", "status")


def shard(n_instances: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous instance block [lo, hi) of `rank` (sizes differ by at most one; ranks
    beyond the instance count get an empty block)."""
    base, rem = divmod(n_instances, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def default_member_instance(n_systems: int, B: int) -> np.ndarray:
    """The member -> instance map DeviceBatch assumes when none is given: one system for
    every member, or one system per member."""
    from .errors import ShapeError
    if n_systems == 1:
        return np.zeros(B, np.int64)
    if n_systems == B:
        return np.arange(B, dtype=np.int64)
    raise ShapeError("member_instance is required when instances != members")


def _row_len(nv: int, trace_len: int | None) -> int:
    return 2 * nv + 6 + (2 * trace_len if trace_len is not None else 0)


def pack(fields: dict, B_pad: int, trace_len: int | None = None):
    """Flatten per-member results into one float64 tensor [B_pad, row] (padded rows = 0).

    Row layout: xi, lam, primal, eq_max, iterations, status, valid flag, global member
    index (fields["index"], default 0..B-1), then the trace if requested."""
    import torch
    B = fields["xi"].shape[0]
    dev = fields["xi"].device
    index = fields.get("index")
    if index is None:
        index = torch.arange(B, dtype=torch.float64, device=dev)
    else:
        index = torch.as_tensor(np.asarray(index), dtype=torch.float64).to(dev)
    parts = [fields["xi"].reshape(B, -1), fields["lam"].reshape(B, -1),
             fields["primal"].reshape(B, 1), fields["eq_max"].reshape(B, 1),
             fields["iterations"].reshape(B, 1).to(torch.float64),
             fields["status"].reshape(B, 1).to(torch.float64),
             torch.ones(B, 1, dtype=torch.float64, device=dev),     # valid flag
             index.reshape(B, 1)]
    if trace_len is not None:
        parts.append(fields["trace"][:, :trace_len].reshape(B, -1))
    flat = torch.cat([p.to(torch.float64) for p in parts], dim=1)
    if B_pad > B:
        flat = torch.cat([flat, flat.new_zeros(B_pad - B, flat.shape[1])])
    return flat.contiguous()


def empty_pack(B_pad: int, nv: int, trace_len: int | None, device):
    """A rank without members sends B_pad padding rows (valid flag 0)."""
    import torch
    return torch.zeros((B_pad, _row_len(nv, trace_len)), dtype=torch.float64, device=device)


def unpack(flat, n_d: int, n: int, n_xi: int, trace_len: int | None = None, order: bool = True) -> dict:
    """Inverse of `pack` on the host: drops padded rows and (order=True) sorts the rows by
    their global member index, so row b is member b of the caller's batch."""
    a = flat.cpu().numpy() if hasattr(flat, "cpu") else np.asarray(flat)
    nv = n_d * n * n_xi
    a = a[a[:, 2 * nv + 4] == 1.0]
    idx = a[:, 2 * nv + 5].astype(np.int64)
    if order:
        perm = np.argsort(idx, kind="stable")
        a, idx = a[perm], idx[perm]
    out = {"xi": a[:, :nv].reshape(-1, n_d, n, n_xi), "lam": a[:, nv:2 * nv].reshape(-1, n_d, n, n_xi),
           "primal": a[:, 2 * nv], "eq_max": a[:, 2 * nv + 1],
           "iterations": a[:, 2 * nv + 2].astype(np.int64), "status": a[:, 2 * nv + 3].astype(np.int64),
           "index": idx}
    if trace_len is not None:
        out["trace"] = a[:, 2 * nv + 6:].reshape(-1, trace_len, 2)
    return out


def _gather_flat(flat, dst: int, group=None):
    import torch
    import torch.distributed as dist
    if flat.is_cuda and dist.get_backend(group) == "gloo":   # gloo gathers host tensors only
        flat = flat.cpu()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [torch.empty_like(flat) for _ in range(world)] if rank == dst else None
    dist.gather(flat, bucket, dst=dst, group=group)
    return None if bucket is None else torch.cat(bucket)


def gather_fields(fields: dict, B_pad: int, dst: int = 0, trace_len: int | None = None, group=None):
    """Gather every rank's packed results to `dst` (NCCL for CUDA tensors, gloo on CPU)."""
    return _gather_flat(pack(fields, B_pad, trace_len), dst, group)


def gather_results(batch, dst: int = 0, B_pad: int | None = None, trace: bool = False, group=None,
                   index=None):
    """Gather a DeviceBatch's results (stream-ordered, no host sync on non-dst ranks).
    `index`: global member index of each of the batch's members (default 0..B-1)."""
    f = {"xi": batch.out_xi, "lam": batch.out_lam, "primal": batch.out_primal,
         "eq_max": batch.out_eq, "iterations": batch.out_its, "status": batch.out_status,
         "index": index}
    T = None
    if trace and batch.out_trace is not None:
        f["trace"] = batch.out_trace
        T = batch.out_trace.shape[1]
    return gather_fields(f, B_pad or batch.B, dst, T, group)


def solve_sharded(systems, xi0, target=None, lam0=None, member_instance=None, kind="projection",
                  cfg=None, fixed_iterations=False, dst=0, trace=False, group=None, cluster=0):
    """Each rank solves the members of its contiguous block of instances; rank `dst`
    returns the full member-major results (dict; row b = member b of the inputs, with
    "trace" (B, max_iters + 1, 2) when trace=True), other ranks None. Inputs are the
    full (global) batch on every rank; a rank whose block is empty solves nothing and
    sends padding only."""
    import torch
    import torch.distributed as dist
    from .solver import DeviceBatch, SolverConfig, system_data
    cfg = cfg or SolverConfig()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    I = len(systems)
    B = int(np.asarray(xi0.shape)[0])
    mi = (default_member_instance(I, B) if member_instance is None
          else np.asarray(member_instance, np.int64))
    blocks = [shard(I, world, r) for r in range(world)]
    lo, hi = blocks[rank]
    sel = np.flatnonzero((mi >= lo) & (mi < hi))
    B_pad = max(1, max(int(np.count_nonzero((mi >= a) & (mi < b))) for a, b in blocks))
    sd = system_data(systems[0], kind, cfg.rho)
    nv = sd.n_d * sd.n * sd.n_basis
    T = cfg.max_iters + 1 if trace else None
    use_cuda = dist.get_backend(group) == "nccl"
    if sel.size == 0:
        dev = torch.device("cuda", torch.cuda.current_device()) if use_cuda else torch.device("cpu")
        flat = _gather_flat(empty_pack(B_pad, nv, T, dev), dst, group)
    else:
        take = lambda x: None if x is None else (x[torch.as_tensor(sel, device=x.device)]
                                                 if isinstance(x, torch.Tensor) else np.asarray(x)[sel])
        batch = DeviceBatch(systems[lo:hi], take(xi0), take(lam0), take(target), kind=kind, cfg=cfg,
                            member_instance=(mi[sel] - lo).astype(np.int32),
                            early_exit=not fixed_iterations, trace=trace, cluster=cluster)
        batch.launch()
        flat = gather_results(batch, dst=dst, B_pad=B_pad, trace=trace, group=group, index=sel)
    if flat is None:
        return None
    out = unpack(flat, sd.n_d, sd.n, sd.n_basis, T)
    assert np.array_equal(out["index"], np.arange(B)), "gather lost or duplicated members"
    return out
