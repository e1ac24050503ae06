"""Top source lines of an `ncu --page source --csv --print-source cuda,sass` export by warp
stall samples.  Usage: python scripts/ncu_source_top.py source.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
lines = []
tot = 0
for r in rows[3:]:
    if len(r) > 4 and r[0] and r[0] != "Line No" and r[1] != "" and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        lines.append((s, r[0], r[1].strip(), r[7]))
        tot += s
lines.sort(reverse=True)
print(f"total samples {tot}")
for s, ln, src, ins in lines[:N]:
    print(f"{100.0 * s / max(tot, 1):5.1f}%  L{ln:>5}  inst={ins:>12}  {src[:110]}")
