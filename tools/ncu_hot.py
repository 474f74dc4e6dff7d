"""Summarise an ncu report's SASS source page: instruction mix and the hottest
instructions by executed count and by stall samples.
    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    ex = lambda r: int(r[ix["Instructions Executed"]] or 0)
    st = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot_ex = sum(ex(r) for r in data)
    tot_st = sum(st(r) for r in data)
    mix = collections.Counter()
    for r in data:
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else op[1]
        mix[o.split(".")[0]] += ex(r)
    print(f"total warp-instructions executed {tot_ex:,}  stall samples {tot_st:,}")
    print("instruction mix (top 25):")
    for o, c in mix.most_common(25):
        print(f"  {o:10s} {c / tot_ex * 100:6.2f}%")
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    for r in data:
        for h in stall_cols:
            agg[h] += int(r[ix[h]] or 0)
    print("stall reasons:", ", ".join(f"{h[6:]} {v / max(tot_st, 1) * 100:.1f}%"
                                      for h, v in agg.most_common(8)))
    print(f"\nhottest by stall samples:")
    for r in sorted(data, key=st, reverse=True)[:top]:
        print(f"  {r[ix['Address']][-5:]} {st(r) / max(tot_st, 1) * 100:5.2f}%  ex={ex(r):>11,}  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main()
