#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/t
R1='(\(int\))?'
XGR_SEED_KERNEL=4 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}5" --launch-skip 1 -c 1 -f -o /tmp/ncu_fused \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/t/fused.log 2>&1; echo "fused rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0" --launch-skip 1 -c 1 -f -o /tmp/ncu_norm \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/t/norm.log 2>&1; echo "norm rc=$?"
for t in fused norm; do
  ncu -i /tmp/ncu_$t.ncu-rep --page source --csv > gpurun_out/t/src_$t.csv 2> gpurun_out/t/src_$t.err
  ncu -i /tmp/ncu_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/t/sass_$t.csv 2> gpurun_out/t/sass_$t.err
done
ls -la gpurun_out/t
