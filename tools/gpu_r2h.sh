#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20" "XGR_DEBUG_FLAGS=16777216::--steps 20" "::--steps 20 --config C2" "XGR_DEBUG_FLAGS=16777216::--steps 20 --config C2" "::--steps 20 --logits bf16" "XGR_STREAM_VARIANT=4::--steps 20 --logits bf16" "XGR_STREAM_VARIANT=5::--steps 20 --logits bf16" "::--steps 10 --config C4" "::--steps 10 --config C5 --split weak" "::--steps 20 --sigma 4" > gpurun_out/ab_h.txt 2>&1
cat gpurun_out/ab_h.txt
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/gputests_h.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_h.log
