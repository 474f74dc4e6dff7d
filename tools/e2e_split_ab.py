"""A/B of the e2e serving loop (solve_stream over the C3 bench batch) with and without the
split schedule: python tools/e2e_split_ab.py [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_09204_b200 import solver  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    systems, xi, mi = bench.make_workload(0)
    cfg = solver.SolverConfig(max_iters=500)
    pin = torch.from_numpy(xi).pin_memory()
    step = (systems, pin, None, pin, mi)
    for label, env in (("split", None), ("nosplit", "1"), ("split", None)):
        if env:
            os.environ["SFB_NO_SPLIT"] = env
        else:
            os.environ.pop("SFB_NO_SPLIT", None)
        for _ in solver.solve_stream(iter([step] * 3), cfg=cfg, fixed_iterations=True):
            pass
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gaps = []
        for _ in solver.solve_stream(iter([step] * steps), cfg=cfg, fixed_iterations=True):
            gaps.append(time.perf_counter())
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(label, "ms/step", round(dt / steps * 1e3, 2), "yield gaps ms",
              [round((b - a) * 1e3, 1) for a, b in zip([t0] + gaps, gaps)], flush=True)


if __name__ == "__main__":
    main()
