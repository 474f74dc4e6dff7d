"""Per-step timeline of the e2e serving loop (solve_stream) on the bench workload:
host time spent building/launching each step, waiting for results, and unpacking them,
next to the device time of each kernel. Explains run-to-run spread of bench.py's `e2e`."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2510_09204_b200 import solver

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 3
systems, xi, mi = bench.make_workload(0)
cfg = solver.SolverConfig(max_iters=bench.WL.get("L", 500))
xi_pin = torch.from_numpy(xi).pin_memory()
step_in = (systems, xi_pin, None, xi_pin, mi)

# instrument: wrap DeviceBatch.__init__ / launch / finish phases
orig_init, orig_launch = solver.DeviceBatch.__init__, solver.DeviceBatch.launch
rec = []
def init(self, *a, **k):
    t = time.perf_counter(); orig_init(self, *a, **k); rec.append(("pack", t, time.perf_counter()))
def launch(self, stream=None):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    s = stream or torch.cuda.current_stream()
    e0.record(s); t = time.perf_counter(); orig_launch(self, stream); rec.append(("launch", t, time.perf_counter()))
    e1.record(s); self._probe = (e0, e1)
solver.DeviceBatch.__init__, solver.DeviceBatch.launch = init, launch

for _ in solver.solve_stream(iter([step_in] * 3), cfg=cfg, fixed_iterations=True, depth=depth):
    pass
torch.cuda.synchronize()
for r in range(reps):
    rec.clear(); kt = []
    t0 = time.perf_counter(); last = t0
    gaps = []
    for res in solver.solve_stream(iter([step_in] * steps), cfg=cfg, fixed_iterations=True, depth=depth):
        now = time.perf_counter(); gaps.append((now - last) * 1e3); last = now
    T = time.perf_counter() - t0
    torch.cuda.synchronize()
    pk = [(b - a) * 1e3 for n, a, b in rec if n == "pack"]
    ln = [(b - a) * 1e3 for n, a, b in rec if n == "launch"]
    print(f"rep {r}: {steps * bench.WL['instances'] / T:7.0f} inst/s  total {T*1e3:7.1f} ms | "
          f"pack ms {np.round(pk, 1).tolist()} | launch ms {np.round(ln, 2).tolist()} | "
          f"yield gaps ms {np.round(gaps, 1).tolist()}", flush=True)
print("loadavg", open("/proc/loadavg").read().strip(), "nproc", os.cpu_count())
