#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20 --config C3Z" "::--steps 20" > gpurun_out/ab_k.txt 2>&1
cat gpurun_out/ab_k.txt
timeout 2400 python -m pytest tests -q -m gpu -x -k "skewed or c3z or topk or random_tries or graph" > gpurun_out/gputests_k.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_k.log
