"""Per-line stall samples and executed warp-instructions of an ncu report, restricted to a
line range of the kernel source (attribution of one stage):
    python tools/ncu_range.py report.ncu-rep FIRST LAST"""
import csv
import io
import subprocess
import sys


def main():
    rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(r for r in rows if "# Samples" in r)
    i_s, i_i = h.index("# Samples"), h.index("Instructions Executed")
    tot_i = 0
    sel = []
    for r in rows[rows.index(h) + 1:]:
        if len(r) == len(h) and r[0]:
            try:
                ln, s, i = int(r[0]), int(r[i_s]), int(r[i_i])
            except ValueError:
                continue
            tot_i += i
            if lo <= ln <= hi:
                sel.append((ln, s, i, r[1].strip()[:110]))
    si = sum(x[2] for x in sel)
    print(f"lines {lo}-{hi}: {si:,} warp-instr ({100 * si / max(tot_i, 1):.1f}%)")
    for ln, s, i, src in sel:
        if i or s:
            print(f"L{ln:<5d} {s:8d} smp {i:14,d} instr  {src}")


if __name__ == "__main__":
    main()
