#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 10 --config C4" "XGR_STREAM_VARIANT=7::--steps 10 --config C4" "::--steps 10 --config C5 --split weak" "XGR_STREAM_VARIANT=7::--steps 10 --config C5 --split weak" > gpurun_out/ab_l.txt 2>&1
cat gpurun_out/ab_l.txt
XGR_STREAM_VARIANT=7 timeout 2400 python -m pytest tests -q -m gpu -x -k "cluster or v16384 or c4_full or c5_full_size_single" > gpurun_out/gputests_l.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_l.log
