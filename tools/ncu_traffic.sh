#!/bin/bash
# One `ncu --set full` capture of the dominant kernel of a bench configuration (one launch, after
# one warm-up pass): gpurun_out/ncu_<tag>.ncu-rep. Usage: tools/ncu_traffic.sh <tag> <kernel regex>
# <bench args...>. Read back here with tools/traffic_json.py.
tag=$1; shift; kre=$1; shift
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$kre" --launch-skip 1 -c 1 -f -o gpurun_out/ncu_$tag \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph "$@" \
  > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"
