#!/bin/bash
# ncu --set full of the latency-bound step kernels of one C3 pass (root k_sparse, seed stream,
# k_seed_theta, k_select, last k_sparse): gpurun_out/ncu_lat_<tag>.ncu-rep. Usage: tools/ncu_latency.sh <tag> [bench args]
tag=$1; shift
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_sparse|k_select|k_seed_theta|k_stream<(\(int\))?32, (\(int\))?1, (\(int\))?2, (\(int\))?3, (\(int\))?3' \
  --launch-skip 5 -c 5 -f -o gpurun_out/ncu_lat_$tag \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph "$@" \
  > gpurun_out/ncu_lat_$tag.log 2>&1
echo "ncu latency $tag rc=$?"
