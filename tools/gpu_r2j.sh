#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 10 --config C5 --split weak" "XGR_DEBUG_FLAGS=8388608::--steps 10 --config C5 --split weak" "XGR_DEBUG_FLAGS=4194304::--steps 10 --config C5 --split weak" "::--steps 10 --config C4" "XGR_DEBUG_FLAGS=8388608::--steps 10 --config C4" "::--steps 20" "XGR_SEED_KERNEL=1::--steps 20" "XGR_SEED_KERNEL=1::--steps 20 --config C2" > gpurun_out/ab_j.txt 2>&1
cat gpurun_out/ab_j.txt
timeout 1800 python -m pytest tests -q -m gpu -x -k "cluster or c4_full or random_tries or v16384" > gpurun_out/gputests_j.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_j.log
