#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20 --config C2" "XGR_THETA_ROWS=4::--steps 20 --config C2" "::--steps 20 --logits bf16" "XGR_THETA_ROWS=4::--steps 20 --logits bf16" "::--steps 20 --sigma 4" "XGR_THETA_ROWS=4::--steps 20 --sigma 4" "::--steps 10 --config C3Z" "XGR_THETA_ROWS=4::--steps 10 --config C3Z" "::--steps 10 --config C4" "XGR_THETA_ROWS=4::--steps 10 --config C4" "::--steps 10 --config C5 --split weak" "XGR_THETA_ROWS=4::--steps 10 --config C5 --split weak" "::--steps 30" "XGR_THETA_ROWS=4::--steps 30" > gpurun_out/ab_u.txt 2>&1
cat gpurun_out/ab_u.txt
