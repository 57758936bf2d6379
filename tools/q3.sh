cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "::--steps 20" "XGR_SEED_MINB=0::--steps 20" "::--steps 20" "XGR_SEED_MINB=0::--steps 20" \
  "::--steps 20 --logits bf16" "XGR_SEED_MINB=0::--steps 20 --logits bf16" "::--steps 20 --config C2" \
  "::--steps 20 --sigma 4" "::--steps 10 --config C4" > gpurun_out/q3_ab.txt 2>&1
cat gpurun_out/q3_ab.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py -q -m gpu -x > gpurun_out/q3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/q3_tests.log
