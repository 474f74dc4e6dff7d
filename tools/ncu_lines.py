"""Summarise an ncu report per CUDA source line (needs -lineinfo and --import-source):
stall samples and executed warp-instructions attributed to each line.
    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(r for r in rows if "# Samples" in r)
    hi = rows.index(h)
    i_s, i_i = h.index("# Samples"), h.index("Instructions Executed")
    data = []
    for r in rows[hi + 1:]:
        if len(r) == len(h) and r[0]:
            try:
                data.append((int(r[i_s]), int(r[i_i]), int(r[0]), r[1].strip()[:100]))
            except ValueError:
                pass
    ts = sum(d[0] for d in data) or 1
    ti = sum(d[1] for d in data) or 1
    print(f"stall samples {ts}, warp-instructions {ti}")
    for s, i, line, src in sorted(data, reverse=True)[:top]:
        print(f"{100 * s / ts:5.1f}% samples {100 * i / ti:5.1f}% instr  L{line:<5d} {src}")


if __name__ == "__main__":
    main()
