cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/q1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/q1/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/q1/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q1/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/q1/default.json 2> gpurun_out/q1/default.err; echo "bench rc=$?"
timeout 600 python bench.py --logits bf16 --no-cpu-baseline --no-e2e > gpurun_out/q1/bf16.json 2> gpurun_out/q1/bf16.err; echo "bench bf16 rc=$?"
