#!/bin/bash
# Source-level ncu captures (--set full --import-source on) for attribution on the dev box:
#   gpurun_out/ncu_src_bf16.ncu-rep : one bf16 C3 k_stream launch (after a warm-up pass)
#   gpurun_out/ncu_src_lat.ncu-rep  : one C3 pass's seed / theta / select / sparse kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
R1='(\(int\))?'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_stream<${R1}32, ${R1}1, ${R1}4, ${R1}3, ${R1}0" --launch-skip 1 -c 1 -f -o gpurun_out/ncu_src_bf16 \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --logits bf16 \
  > gpurun_out/ncu_src_bf16.log 2>&1
echo "ncu bf16 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_seed_hist|k_seed_theta|k_select|k_sparse' --launch-skip 5 -c 5 -f -o gpurun_out/ncu_src_lat \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph \
  > gpurun_out/ncu_src_lat.log 2>&1
echo "ncu lat rc=$?"
ls -la gpurun_out/*.ncu-rep
