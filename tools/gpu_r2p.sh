#!/bin/bash
# fused seed (XGR_SEED_KERNEL=4): parity first, then A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
XGR_SEED_KERNEL=4 timeout 900 python -m pytest tests -q -m gpu -x -k "random_tries or c2_full or c3_full or skewed or pruning or smoke" > gpurun_out/gputests_p.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_p.log
bash tools/ab.sh "::--steps 20" "XGR_SEED_KERNEL=4::--steps 20" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=4::--steps 20" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=12::--steps 20" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=16::--steps 20" "XGR_THETA_ROWS=4::--steps 20" "::--steps 20 --config C2" "XGR_SEED_KERNEL=4::--steps 20 --config C2" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=4::--steps 20 --config C2" "::--steps 10 --config C3Z" "XGR_SEED_KERNEL=4::--steps 10 --config C3Z" "::--steps 20 --sigma 4" "XGR_SEED_KERNEL=4::--steps 20 --sigma 4" > gpurun_out/ab_p.txt 2>&1
cat gpurun_out/ab_p.txt
