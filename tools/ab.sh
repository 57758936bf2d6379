# A/B timing helper (diagnostic): runs the default bench for each env setting given as args
for v in "$@"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --no-e2e > "gpurun_out/ab_${v// /_}.json" 2>/dev/null
done
