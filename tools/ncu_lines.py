"""Aggregate an ncu source page (cuda,sass CSV) per source line: share of warp
stall samples, top stall reasons, excessive shared wavefronts.
usage: ncu -i REP --page source --csv --print-source cuda,sass --launch-skip K --launch-count 1 > x.csv
       python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None
out = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if hdr and r and r[0].isdigit() and len(r) > 6:
        try:
            s = float(r[6] or 0)
        except ValueError:
            continue
        if s > 0:
            out.append((s, cur, int(r[0]), r[1][:80], r))
tot = sum(o[0] for o in out)
ix = {k: i for i, k in enumerate(hdr)}
for s, f, l, src, r in sorted(out, reverse=True)[:top]:
    st = sorted([(float(r[i] or 0), k) for k, i in ix.items() if k.startswith("stall_") and "Not" not in k],
                reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}% {f}:{l} {src}  {[(k[6:], round(v / tot * 100, 1)) for v, k in st]} "
          f"wfex={r[ix['L1 Wavefronts Shared Excessive']]}")
