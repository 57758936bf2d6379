#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_m.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_m.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/gputests_m.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_m.log
timeout 900 python bench.py --config C5 --split weak --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/final_C5w.json 2> gpurun_out/final_C5w.err; echo "C5w rc=$?"
