#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NR=$PWD/paper_2512_11529_b200/lib/libxgr_beam_norot.so
bash tools/ab.sh "::--steps 20" "XGR_LIB=$NR::--steps 20" "::--steps 20" "XGR_LIB=$NR::--steps 20" "::--steps 10 --config C4" "XGR_LIB=$NR::--steps 10 --config C4" "::--steps 10 --config C5 --split weak" "XGR_LIB=$NR::--steps 10 --config C5 --split weak" "XGR_STREAM_VARIANT=6::--steps 10 --config C5 --split weak" "::--steps 20 --config C2" > gpurun_out/ab_i.txt 2>&1
cat gpurun_out/ab_i.txt
timeout 2400 python -m pytest tests -q -m gpu -x -k "random_tries or c1 or c2_full or cluster or pruning or shard or topk or bf16 or graph or v16384 or skewed or paper_heap or head" > gpurun_out/gputests_i.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_i.log
