#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20" "XGR_DEBUG_FLAGS=8388608::--steps 20" "::--steps 20" "XGR_DEBUG_FLAGS=8388608::--steps 20" "::--steps 20 --logits bf16" "XGR_DEBUG_FLAGS=8388608::--steps 20 --logits bf16" "::--steps 10 --config C4" "XGR_DEBUG_FLAGS=8388608::--steps 10 --config C4" "::--steps 20 --paper-heap --no-graph" > gpurun_out/ab_sleep.txt 2>&1
cat gpurun_out/ab_sleep.txt
timeout 1500 python -m pytest tests -q -m gpu -x -k "paper_heap or request_split" > gpurun_out/gputests_f.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_f.log
bash tools/ncu_traffic.sh C4_f32 'k_stream<(\(int\))?32, (\(int\))?1, (\(int\))?2, (\(int\))?3, (\(int\))?0, float, (\(int\))?256, (\(int\))?2' --config C4
bash tools/ncu_traffic.sh C3Z_f32 'k_stream<(\(int\))?32, (\(int\))?1, (\(int\))?2, (\(int\))?3, (\(int\))?0, float, (\(int\))?256, (\(int\))?1' --config C3Z
bash tools/ncu_traffic.sh C5_f32 'k_stream<(\(int\))?32, (\(int\))?1, (\(int\))?2, (\(int\))?3, (\(int\))?0, float, (\(int\))?256, (\(int\))?8' --config C5 --split weak
