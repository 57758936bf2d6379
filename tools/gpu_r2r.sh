#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
F="XGR_SEED_KERNEL=4"
bash tools/ab.sh "$F::--steps 20" "$F XGR_DEBUG_FLAGS=33554432::--steps 20" "$F XGR_DEBUG_FLAGS=67108864::--steps 20" "$F XGR_DEBUG_FLAGS=100663296::--steps 20" "$F XGR_DEBUG_FLAGS=134217728::--steps 20" "$F XGR_DEBUG_FLAGS=268435456::--steps 20" "$F XGR_THETA_ROWS=1::--steps 20" "$F XGR_THETA_ROWS=2::--steps 20" "XGR_THETA_ROWS=2::--steps 20" "XGR_THETA_ROWS=3::--steps 20" "XGR_THETA_ROWS=4::--steps 20" "XGR_THETA_ROWS=5::--steps 20" "XGR_THETA_ROWS=6::--steps 20" "::--steps 20" > gpurun_out/ab_r.txt 2>&1
cat gpurun_out/ab_r.txt
