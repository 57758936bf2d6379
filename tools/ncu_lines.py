"""Aggregate an ncu source page (--print-source sass,cuda --csv) to CUDA source lines:
stall samples and executed warp instructions per line. Usage: python tools/ncu_lines.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = {}
fname = None
cur_line = None
cur_src = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    # rows: line-no, cuda source, address, sass, samples, not-issued, #samples, inst executed, ...
    if r[0]:
        cur_line = (fname, int(r[0]))
        cur_src = r[1]
    if len(r) > 7 and r[2]:
        try:
            w = int(r[4] or 0)
            n = int(r[7] or 0)
        except ValueError:
            continue
        a = agg.setdefault(cur_line, [0, 0, cur_src])
        a[0] += w
        a[1] += n
tw = sum(v[0] for v in agg.values()) or 1
tn = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tw}, warp instructions {tn}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tw * 100:5.1f}% stall {v[1] / tn * 100:5.1f}% inst  {k[0]}:{k[1]:<5d} {v[2].strip()[:70]}")
