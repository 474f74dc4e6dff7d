"""Time the trajectory-metrics epilogue (sfb_trajectory_metrics) on the C3 workload's 512
members (64 instances x 8 candidates, 32 robots, 20 obstacles, 10x dense grid = 991 points),
device-resident inputs, CUDA events; and the oracle (numpy restatement of metrics.py:48-87)
on a few members on one host core. Writes profiles/r01_metrics.json.

    python tools/bench_metrics.py [--members 512] [--reps 20]
"""

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.metrics import trajectory_metrics  # noqa: E402
from paper_2510_09204_b200 import _lib, metrics as M  # noqa: E402
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, build_basis, generate,  # noqa: E402
                                           sample_naive_prior, stack_xi)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=512)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    cfg = BasisConfig(11, 100, 5.0)
    basis = build_basis(cfg)
    scn = generate(ScenarioFamily("random_box", box=(-2.0, 2.0), n_obstacles=20), 32, 2, seed=3000,
                   horizon=cfg)
    xi = stack_xi(sample_naive_prior(scn, basis, a.members, seed=1))
    mm = np.ascontiguousarray(xi.reshape(2, 32, 11, a.members).transpose(3, 0, 1, 2))
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(mm).to(dev)
    ref = M.metrics_batch(x, basis, scn)                          # warm + result
    dense = M.dense_basis(basis)
    obs, _ = M._obstacle_array(scn, 2, a.members)
    host = [np.ascontiguousarray(v, float).ravel() for v in (basis.Wdd, dense.W, dense.grid, obs)]
    offs = np.cumsum([0] + [v.size for v in host])
    consts = torch.from_numpy(np.concatenate(host)).to(dev)
    L = _lib.lib()
    B, kd = a.members, dense.W.shape[0]
    nwork = L.sfb_trajectory_metrics_work(B, 2, 32, 11, kd, obs.shape[0])
    scratch = torch.empty(nwork + B * 5, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    p = lambda k: consts.data_ptr() + 8 * int(offs[k])  # noqa: E731

    def launch():
        rc = L.sfb_trajectory_metrics(x.data_ptr(), B, 2, 32, 11, p(0), basis.Wdd.shape[0], p(1), p(2),
                                      kd, p(3), obs.shape[0], 0, scratch.data_ptr(),
                                      scratch.data_ptr() + 8 * nwork, ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "metrics")

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        launch()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    got = scratch[nwork:].view(B, 5).cpu().numpy()
    assert np.array_equal(got, ref)
    ob = [(o.center, o.velocity, o.radii) for o in scn.obstacles]
    t = time.perf_counter()
    ncpu = 4
    for k in range(ncpu):
        o = trajectory_metrics(mm[k].transpose(1, 0, 2), 11, 100, 5.0, ob, 10)
        assert np.all(np.abs(o - ref[k]) <= 1e-12 * np.maximum(1, np.abs(o)))
    cpu_ms = (time.perf_counter() - t) * 1e3 / ncpu
    n, m = 32, 20
    pairs = n * (n - 1) // 2 * kd
    terms = pairs + m * n * kd + n * (kd - 1) + n * 100
    res = {"workload": "C3 metrics epilogue (metrics.py:48-87), 10x dense grid", "members": B,
           "dense_points": kd, "distance_terms_per_member": terms, "ms_per_batch": ms,
           "members_per_s": B / ms * 1e3, "gterms_per_s": terms * B / ms / 1e6,
           "cpu_oracle_ms_per_member_1core": cpu_ms, "cpu_members_per_s_1core": 1e3 / cpu_ms}
    print(json.dumps(res))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "metrics.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
