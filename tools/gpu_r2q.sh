#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20" "XGR_SEED_KERNEL=4::--steps 20" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=4::--steps 20" "XGR_SEED_KERNEL=4 XGR_THETA_ROWS=16::--steps 20" "::--steps 20 --config C2" "XGR_SEED_KERNEL=4::--steps 20 --config C2" > gpurun_out/ab_q.txt 2>&1
cat gpurun_out/ab_q.txt
XGR_SEED_KERNEL=4 timeout 900 python -m pytest tests -q -m gpu -x -k "random_tries or c2_full or c3_full or pruning" > gpurun_out/gputests_q.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_q.log
