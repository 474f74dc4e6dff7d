"""The N > 1 path on one GPU (the round's GPU box has one): two ranks share cuda:0 over gloo
and run parallel.solve_sharded — contiguous instance shards, each rank's DeviceBatch on the
GPU, one gather of the final results (trace included) to rank 0. Rank 0's gathered results
must be bitwise those of one process solving the whole batch (the members
never interact). NCCL refuses two ranks on one device, so the gather itself runs over gloo
here; the NCCL path is the same gather call (parallel._gather_flat) on CUDA tensors."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _workload():
    from paper_2510_09204_b200 import solver
    from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble, build_basis,
                                               generate, sample_naive_prior, stack_xi)
    basis = build_basis(BasisConfig(11, 100, 5.0))
    fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-2.0, 2.0), n_obstacles=20)
    systems, xs = [], []
    for i in range(5):
        scn = generate(fam, 32, 2, seed=7000 + i, horizon=basis.config)
        systems.append(assemble(scn, basis))
        xs.append(solver.to_member_major(stack_xi(sample_naive_prior(scn, basis, 3, seed=7000 + i)), 32, 11))
    mi = np.tile(np.arange(5), 3)                     # interleaved member -> instance map
    xi = np.stack([xs[b % 5][b // 5] for b in range(15)])   # member b = sample b // 5 of instance b % 5
    return systems, xi, mi


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_09204_b200 import parallel, solver
    systems, xi, mi = _workload()
    cfg = solver.SolverConfig(max_iters=40)
    out = parallel.solve_sharded(systems, xi, target=xi, member_instance=mi, cfg=cfg,
                                 fixed_iterations=True, trace=True, cluster=1)
    if rank == 0:
        q.put({k: out[k] for k in ("xi", "lam", "primal", "eq_max", "iterations", "status", "trace", "index")})
    dist.barrier()
    dist.destroy_process_group()


def test_solve_sharded_two_ranks_bitwise_equals_one_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    from paper_2510_09204_b200 import solver
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    systems, xi, mi = _workload()
    cfg = solver.SolverConfig(max_iters=40)
    ref = solver.solve_instances(systems, xi, None, xi, member_instance=mi.astype(np.int32), cfg=cfg,
                                 fixed_iterations=True, trace=True, cluster=1)
    assert np.array_equal(got["index"], np.arange(len(xi)))
    assert np.array_equal(got["xi"], ref.xi) and np.array_equal(got["lam"], ref.lam)
    assert np.array_equal(got["primal"], ref.primal) and np.array_equal(got["eq_max"], ref.eq_violation_max)
    assert np.array_equal(got["iterations"], ref.iterations)
    for b in range(len(xi)):
        assert np.array_equal(got["trace"][b], ref.trace[b])
