"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a bench.py --profile run:
every xgr kernel launch in order, then per-kernel totals and shares of the timed passes.
Usage: python tools/launch_shares.py launches.csv > profiles/<name>_launches_xgr.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
launches = []
for r in rows[1:]:
    if "xgr" not in r[ki] or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v * 1000.0 if r[ui] == "usecond" else v
    name = r[ki].split("(")[0].replace("void ", "")
    launches.append((name, v))
print("# ncu --metrics gpu__time_duration.sum --clock-control none: every xgr kernel launch of")
print("# `python bench.py --profile --steps 2 --warmup 1 --no-e2e` (setup, 1 warm-up + 2 timed passes,")
print("# accounting pass); cold-cache, serialised launches: compare SHARES, not absolutes")
for n, v in launches:
    print(f"{n:48s} {v:12.0f} ns")
STEP = ("k_stream", "k_seed", "k_select", "k_sparse", "k_main", "k_theta", "k_merge")
step_kernels = [(n, v) for n, v in launches if any(k in n for k in STEP)]
tot = collections.OrderedDict()
for n, v in step_kernels:
    tot[n] = tot.get(n, 0.0) + v
s = sum(tot.values())
print("\n# per-kernel totals over the decode passes (warm-up + timed), share of the pass")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{n:48s} {v / 1000:10.1f} us  {100 * v / s:5.1f}%")
