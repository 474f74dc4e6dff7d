"""Attribute an ncu report's executed warp-instructions and stall samples to kernel
stages (line ranges of csrc/sfb_kernel.cuh). SASS inlined from CUDA headers is charged
to the stage of the nearest preceding kernel-file instruction (by address).
    python tools/ncu_regions.py report.ncu-rep"""
import bisect
import csv
import io
import re
import subprocess
import sys

def stages(path):
    """(first line, name) markers: a line containing `// @stage name` starts a stage."""
    out = []
    with open(path) as fh:
        for no, line in enumerate(fh, 1):
            m = re.search(r"//\s*@stage\s+(\S+)", line)
            if m:
                out.append((no, m.group(1)))
    return out


def main():
    rep = sys.argv[1]
    kpath = sys.argv[2] if len(sys.argv) > 2 else "paper_2510_09204_b200/csrc/sfb_kernel.cuh"
    kfile = kpath.rsplit("/", 1)[-1]
    marks = stages(kpath)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file, cur_line, hdr = None, None, None
    insts = []   # (addr, file, line, executed, samples)
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0]:
            try:
                cur_line = int(r[0])
            except ValueError:
                pass
            continue
        addr = r[2]
        try:
            wf = int(r[hdr.index("L1 Wavefronts Shared")] or 0)
            wi = int(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
            insts.append((int(addr, 16), cur_file, cur_line, int(r[7] or 0), int(r[6] or 0), wf, wi))
        except ValueError:
            pass
    insts.sort()
    lines_sorted = [m[0] for m in marks]
    agg = {}
    last_stage = "prologue"
    for addr, f, line, ex, sm, wf, wi in insts:
        if f and f.endswith(kfile) and line is not None:
            k = bisect.bisect_right(lines_sorted, line) - 1
            last_stage = marks[k][1] if k >= 0 else "prologue"
        e = agg.setdefault(last_stage, [0, 0, 0, 0])
        e[0] += ex
        e[1] += sm
        e[2] += wf
        e[3] += wi
    te = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    tw = sum(v[2] for v in agg.values()) or 1
    print(f"{'stage':24s} {'instr %':>8s} {'stall %':>8s} {'smem wf %':>9s} {'wf/ideal':>8s}   warp-instr")
    order = [m[1] for m in marks]
    for name in ["prologue"] + order:
        if name in agg:
            e, s, w, wi = agg.pop(name)
            print(f"{name:24s} {100 * e / te:8.1f} {100 * s / ts:8.1f} {100 * w / tw:9.1f} "
                  f"{(w / wi if wi else 0):8.2f}   {e:,}")
    print(f"total shared-memory wavefronts {tw:,}")


if __name__ == "__main__":
    main()
