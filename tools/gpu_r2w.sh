#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20 --logits bf16" "XGR_STREAM_VARIANT=10::--steps 20 --logits bf16" "::--steps 20" "XGR_STREAM_VARIANT=11::--steps 20" "::--steps 20 --config C2" "XGR_STREAM_VARIANT=11::--steps 20 --config C2" "::--steps 20 --config C2 --logits bf16" "XGR_STREAM_VARIANT=10::--steps 20 --config C2 --logits bf16" > gpurun_out/ab_w.txt 2>&1
cat gpurun_out/ab_w.txt
XGR_STREAM_VARIANT=10 timeout 900 python -m pytest tests/test_gpu_bf16.py -q -x > gpurun_out/gputests_w.log 2>&1; echo "bf16 tests v10 rc=$?"; tail -2 gpurun_out/gputests_w.log
