"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 path: contiguous
instance shards and the single gather of final results to rank 0
(paper_2510_09204_b200/parallel.py)."""

import os
import socket

import numpy as np
import pytest

from paper_2510_09204_b200 import parallel

torch = pytest.importorskip("torch")


def test_shard_covers_instances_contiguously():
    for I in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            blocks = [parallel.shard(I, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == I
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c and b - a >= d - c
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def test_pack_unpack_round_trip():
    B, nd, n, nxi, T = 5, 2, 3, 4, 6
    g = torch.Generator().manual_seed(0)
    f = {"xi": torch.randn(B, nd, n, nxi, generator=g, dtype=torch.float64),
         "lam": torch.randn(B, nd, n, nxi, generator=g, dtype=torch.float64),
         "primal": torch.rand(B, dtype=torch.float64), "eq_max": torch.rand(B, dtype=torch.float64),
         "iterations": torch.arange(B, dtype=torch.int32), "status": torch.ones(B, dtype=torch.int32),
         "trace": torch.randn(B, T, 2, dtype=torch.float64)}
    flat = parallel.pack(f, 8, T)
    assert flat.shape[0] == 8
    out = parallel.unpack(flat, nd, n, nxi, T)
    assert out["xi"].shape[0] == B
    for k in ("xi", "lam", "primal", "eq_max", "trace"):
        assert np.array_equal(out[k], f[k].numpy())
    assert np.array_equal(out["iterations"], np.arange(B))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B = 3 if rank == 0 else 2           # unequal shards -> padding
    f = {"xi": torch.full((B, 2, 2, 4), float(rank), dtype=torch.float64),
         "lam": torch.full((B, 2, 2, 4), -float(rank), dtype=torch.float64),
         "primal": torch.arange(B, dtype=torch.float64) + 10 * rank,
         "eq_max": torch.zeros(B, dtype=torch.float64),
         "iterations": torch.full((B,), 500 + rank, dtype=torch.int32),
         "status": torch.zeros(B, dtype=torch.int32),
         "index": np.arange(B) + (0 if rank == 0 else 3)}
    flat = parallel.gather_fields(f, B_pad=3, dst=0)
    if rank == 0:
        out = parallel.unpack(flat, 2, 2, 4)
        q.put((out["xi"][:, 0, 0, 0].tolist(), out["primal"].tolist(), out["iterations"].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_to_rank0_gloo_world2():
    import multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    xi0, primal, its = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert xi0 == [0.0, 0.0, 0.0, 1.0, 1.0]
    assert primal == [0.0, 1.0, 2.0, 10.0, 11.0]
    assert its == [500, 500, 500, 501, 501]


# ------------------------------------------------------------ solve_sharded host logic
class _FakeBatch:
    """Stands in for DeviceBatch in the CPU test: 'solves' member b of local instance
    k by returning xi = xi0 + 1000 * (global instance) and iterations = global instance,
    so the gathered rows say which rank solved which member."""

    lo = 0

    def __init__(self, systems, xi0, lam0, target, kind, cfg, member_instance, early_exit, trace,
                 cluster=0):
        mi = torch.as_tensor(np.asarray(member_instance, np.int64))
        inst = (mi + _FakeBatch.lo).to(torch.float64)
        x = torch.as_tensor(np.asarray(xi0, float))
        self.B = x.shape[0]
        self.out_xi = x + 1000.0 * inst.view(-1, 1, 1, 1)
        self.out_lam = -self.out_xi
        self.out_primal = inst.clone()
        self.out_eq = torch.zeros(self.B, dtype=torch.float64)
        self.out_its = inst.to(torch.int32)
        self.out_status = torch.zeros(self.B, dtype=torch.int32)
        T = cfg.max_iters + 1
        self.out_trace = inst.view(-1, 1, 1).expand(self.B, T, 2).clone() if trace else None

    def launch(self, stream=None):
        pass


def _sharded_worker(rank, world, port, q, n_inst, samples, interleave):
    import torch.distributed as dist
    from paper_2510_09204_b200 import solver
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import golden_io
    g = golden_io.load("obs8_projection")
    d = g.sys.dims
    systems = [g.sys] * n_inst
    B = n_inst * samples
    mi = (np.tile(np.arange(n_inst), samples) if interleave
          else np.repeat(np.arange(n_inst), samples))
    xi0 = np.random.default_rng(0).standard_normal((B, d.n_d, d.n, d.n_basis))
    _FakeBatch.lo = parallel.shard(n_inst, world, rank)[0]
    orig = solver.DeviceBatch
    solver.DeviceBatch = _FakeBatch
    try:
        out = parallel.solve_sharded(systems, xi0, target=xi0, member_instance=mi,
                                     cfg=solver.SolverConfig(max_iters=3), fixed_iterations=True,
                                     trace=True)
    finally:
        solver.DeviceBatch = orig
    if rank == 0:
        ok_xi = np.array_equal(out["xi"], xi0 + 1000.0 * mi[:, None, None, None])
        q.put((ok_xi, out["iterations"].tolist(), mi.tolist(), out["trace"][:, -1, 0].tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_inst,samples,interleave", [(3, 2, True), (1, 3, False), (4, 2, True)])
def test_solve_sharded_order_and_empty_ranks_gloo_world2(n_inst, samples, interleave):
    """interleaved member->instance maps come back in the caller's member order,
    and a rank without instances (I < world) sends padding only."""
    import multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, n_inst, samples, interleave))
             for r in range(2)]
    for p in procs:
        p.start()
    ok_xi, its, mi, tr = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok_xi
    assert its == mi and tr == [float(v) for v in mi]


def test_default_member_instance():
    assert parallel.default_member_instance(1, 3).tolist() == [0, 0, 0]
    assert parallel.default_member_instance(3, 3).tolist() == [0, 1, 2]
    from paper_2510_09204_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        parallel.default_member_instance(2, 3)
