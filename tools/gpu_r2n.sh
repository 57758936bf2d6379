#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 10 --config C4" "XGR_STREAM_VARIANT=9::--steps 10 --config C4" "::--steps 10 --config C5 --split weak" "XGR_STREAM_VARIANT=9::--steps 10 --config C5 --split weak" > gpurun_out/ab_n.txt 2>&1
cat gpurun_out/ab_n.txt
