#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_boundary.py -q -x > gpurun_out/gputests_v.log 2>&1; echo "boundary rc=$?"; tail -30 gpurun_out/gputests_v.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_v.log
timeout 600 python bench.py --steps 10 > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
