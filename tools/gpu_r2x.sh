#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/x
timeout 1500 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -x -k "boundary or host or alloc or fused" > gpurun_out/x/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/x/tests.log
timeout 600 python tools/sanitize_fused.py > gpurun_out/x/plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/x/plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_fused.py > gpurun_out/x/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/x/san_$tool.log
done
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_boundary.py -q -x -k "alloc or host_logits_step" > gpurun_out/x/san_boundary.log 2>&1; echo "boundary memcheck rc=$?"; tail -3 gpurun_out/x/san_boundary.log
