#!/bin/bash
# ncu --set full of the fused-seed k_stream vs the default one (C3), summarised on the box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/s
R1='(\(int\))?'
XGR_SEED_KERNEL=4 timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
  -k "regex:k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}5" --launch-skip 1 -c 1 -f -o /tmp/ncu_fused \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/s/fused.log 2>&1; echo "fused rc=$?"
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
  -k "regex:k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0" --launch-skip 1 -c 1 -f -o /tmp/ncu_norm \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/s/norm.log 2>&1; echo "norm rc=$?"
for t in fused norm; do
  ncu -i /tmp/ncu_$t.ncu-rep --page raw --csv > /tmp/raw_$t.csv 2>/dev/null
  python - /tmp/raw_$t.csv > gpurun_out/s/$t.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
for r in rows[2:]:
    for i, name in enumerate(h):
        if any(k in name for k in ("stalled", "time_duration", "dram__bytes", "inst_executed.sum", "issue_active", "warps_active", "cycles_elapsed.max", "Kernel Name")):
            print(f"{name:90s} {r[i]} {u[i]}")
PY
done
head -c 20000 gpurun_out/s/fused.txt | grep -i "duration\|sleep\|membar\|long_score\|barrier_per\|inst_executed.sum \|dram__bytes_read.sum \|wait_per\|branch\|lg_thr\|no_inst\|mio"
echo ----
grep -i "duration\|sleep\|membar\|long_score\|barrier_per\|inst_executed.sum \|dram__bytes_read.sum \|wait_per\|branch\|lg_thr\|no_inst\|mio" gpurun_out/s/norm.txt
