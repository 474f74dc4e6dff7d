"""Write the committed profile summaries of one measurement run into profiles/:
    python tools/save_profiles.py <tag> <full .ncu-rep> <launch-list csv> [bench json] [ref json]
-> profiles/<tag>_ncu_details.csv, <tag>_ncu_hot.txt, <tag>_launches_summary.txt,
   <tag>_bench_line.json, <tag>_bench_reference_line.json, ncu_traffic.json (read by bench.py)."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def run(*cmd):
    return subprocess.run(list(cmd), capture_output=True, text=True).stdout


def main():
    tag, rep, launches = sys.argv[1:4]
    py = sys.executable
    with open(os.path.join(PROF, f"{tag}_ncu_details.csv"), "w") as fh:
        fh.write(run("ncu", "-i", rep, "--page", "details", "--csv"))
    reg = run(py, os.path.join(ROOT, "tools", "ncu_regions.py"), rep)
    hot = run(py, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "30")
    lines = run(py, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "40")
    with open(os.path.join(PROF, f"{tag}_ncu_hot.txt"), "w") as fh:
        fh.write("ncu --set full --clock-control none --import-source on -k regex:sf_solve -s 1 -c 1 "
                 "tools/profile_c3.py 2 (C3 batch, 512 members x 501 evals)\n\n"
                 "== per kernel stage (tools/ncu_regions.py; smem wf = shared-memory wavefronts)\n"
                 + reg + "\n== SASS (tools/ncu_hot.py)\n" + hot + "\n== per CUDA source line (tools/ncu_lines.py)\n"
                 + lines)
    # launch list
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) == len(h) and r[mn] == "gpu__time_duration.sum":
            a = agg[r[kn]]
            a[0] += 1
            a[1] += float(r[mv].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none on "
           "`bench.py --steps 2 --warmup 1 --no-cpu --latency 0`",
           "(cold-cache, serialised replays: compare shares, not absolutes)", ""]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{100 * t / tot:6.2f}%  n={n:4d}  total={t:14.0f} ns  {k[:90]}")
    with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    # DRAM traffic of the captured launch
    raw = list(csv.reader(run("ncu", "-i", rep, "--page", "raw", "--csv").splitlines()))
    hdr, unit, val = raw[0], raw[1], raw[2]
    def metric(name):
        v = float(val[hdr.index(name)].replace(",", ""))
        u = unit[hdr.index(name)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}.get(u, 1)
        return v * scale
    rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as fh:
        json.dump({"kernel": "sf_solve_kernel<2,11,32,0> (C3 batch, 512 members x 501 evals)",
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                   "gpu_time_ms": metric("gpu__time_duration.sum"),
                   "source": f"ncu --set full --clock-control none ({tag}_ncu_details.csv)"}, fh, indent=1)
    if len(sys.argv) > 4:
        shutil.copy(sys.argv[4], os.path.join(PROF, f"{tag}_bench_line.json"))
    if len(sys.argv) > 5:
        shutil.copy(sys.argv[5], os.path.join(PROF, f"{tag}_bench_reference_line.json"))


if __name__ == "__main__":
    main()
