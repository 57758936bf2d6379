cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
H=XGR_LIB=$PWD/paper_2512_11529_b200/lib/ab/head.so
bash tools/ab.sh "$H::--steps 30" "::--steps 30" "$H::--steps 30" "::--steps 30" "$H::--steps 30" "::--steps 30" \
  "$H::--steps 20 --logits bf16" "::--steps 20 --logits bf16" "$H::--steps 20 --config C2" "::--steps 20 --config C2" \
  "$H::--steps 10 --config C4" "::--steps 10 --config C4" > gpurun_out/q4_ab.txt 2>&1
cat gpurun_out/q4_ab.txt
for v in head new; do
  if [ $v = head ]; then export XGR_LIB=$PWD/paper_2512_11529_b200/lib/ab/head.so; else unset XGR_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/q4_launch_$v.csv \
    python bench.py --profile --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch $v rc=$?"
done
unset XGR_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_topk.py tests/test_gpu_skewed.py tests/test_gpu_graph.py -q -m gpu -x > gpurun_out/q4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/q4_tests.log
