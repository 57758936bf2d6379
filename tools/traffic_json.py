"""Writes profiles/ncu_k_stream_<cfg>_<dtype>[_s<sigma>]_traffic.json (the roofline `traffic` of
bench.py) and a metric summary from one `ncu --set full` capture (tools/ncu_traffic.sh).
Usage: python tools/traffic_json.py <report.ncu-rep> <cfg> <dtype> <sigma> <round tag>"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, cfg, dtype, sigma, tag = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5]
OUT = sys.argv[6] if len(sys.argv) > 6 else ROOT   # on the GPU box: a directory under gpurun_out/
SPLIT = sys.argv[7] if len(sys.argv) > 7 else ""     # a non-default partition (e.g. "weak" for C5)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, r = rows[0], rows[1], rows[2]


def val(m):
    v = float(r[hdr.index(m)].replace(",", ""))
    u = units[hdr.index(m)]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
summary = os.path.join("profiles", f"{tag}_ncu_{cfg}{'_' + SPLIT if SPLIT else ''}_{dtype}{'' if sigma == 2.0 else f'_s{sigma:g}'}.txt")
out = {"kernel": r[hdr.index("Kernel Name")][:160], "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
       "duration_ns_under_ncu": val("gpu__time_duration.sum"),
       "source": f"{summary} (ncu --set full --clock-control none, one launch after a warm-up pass)"}
os.makedirs(os.path.join(OUT, "profiles"), exist_ok=True)
with open(os.path.join(OUT, "profiles", bench.traffic_key(cfg, dtype, sigma, SPLIT)), "w") as f:
    json.dump(out, f, indent=1)
s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                   text=True, check=True).stdout
with open(os.path.join(OUT, summary), "w") as f:
    f.write(f"# {rep}: bench.py --config {cfg} --logits {dtype} --sigma {sigma:g}, dominant kernel\n" + s)
print(json.dumps(out))
