#!/bin/bash
# One `ncu --set full` capture of the dominant kernel of a bench configuration (one launch, after
# one warm-up pass), summarised on the box (tools/traffic_json.py) into
# gpurun_out/final/profiles/{ncu_k_stream_*_traffic.json, <round>_ncu_<cfg>.txt}; the report itself
# stays in /tmp (gpurun_out/ is capped at 64 MiB) unless KEEP_REP=1.
# LSKIP=<n>: matching launches to skip (default 1: the warm-up pass's first).
# Usage: tools/ncu_traffic.sh <tag> <kernel regex> <cfg> <dtype> <sigma> <split|-> <bench args...>
tag=$1; kre=$2; cfg=$3; dt=$4; sg=$5; sp=$6; shift 6
[ "$sp" = "-" ] && sp=""
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
rep=/tmp/ncu_$tag
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$kre" --launch-skip ${LSKIP:-1} -c 1 -f -o $rep \
  python bench.py --profile --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph "$@" \
  > gpurun_out/final/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"
python tools/traffic_json.py $rep.ncu-rep $cfg $dt $sg r02 gpurun_out/final $sp > gpurun_out/final/traffic_$tag.log 2>&1
[ "${KEEP_REP:-0}" = "1" ] && cp $rep.ncu-rep gpurun_out/final/
true
