"""Per-phase cycle breakdown of the C3 solve (needs a libsfb.so built with
-DSFB_PHASE_TIMING; SFB_LIB points to it)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2510_09204_b200 import solver

systems, xi, mi = bench.make_workload(0)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 500
n_inst = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cluster = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sel = mi < n_inst
systems, xi, mi = systems[:n_inst], xi[sel], mi[sel]
batch = solver.DeviceBatch(systems, xi, None, xi, cfg=solver.SolverConfig(max_iters=L),
                           member_instance=mi, early_exit=False, trace=False, counters=True,
                           cluster=cluster)
batch.out_counters = torch.zeros((batch.B, 24), dtype=torch.int64, device=batch.device)
batch._build_structs()
batch.launch(); torch.cuda.synchronize()
batch.launch(); torch.cuda.synchronize()
c = batch.out_counters.cpu().numpy().astype(float)
names = ["tasks", "bar_after_tasks", "G_reduce", "decision", "K1+bar", "K2+K3+bar"]
sub_names = ["  positions", "  robot screen", "  robot exact", "  obstacles", "  box+contract",
             "  cluster.sync", "  dsmem reads", "  post-read bar", "  E2 mean", "  E2 dmma+store",
             "  G contraction (own tile)", "  E1 columns (own)"]
per = c[:, 4:10].mean(axis=0) / (L + 1)
sub = c[:, 10:22].mean(axis=0) / (L + 1)
tot = per.sum()
for nm, v in zip(names, per):
    print(f"{nm:18s} {v:9.0f} cycles/iter ({v / tot * 100:5.1f}%)")
print(f"total {tot:.0f} cycles/iter per CTA = {tot / 1.965e3:.2f} us")
for nm, v in zip(sub_names, sub):
    print(f"{nm:18s} {v:9.0f} cycles/iter (warp 0)")
