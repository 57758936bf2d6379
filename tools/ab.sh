# A/B timing helper (diagnostic). Each argument is "ENV=V ENV2=V2::bench args"; the bench JSON of
# each goes to gpurun_out/ab_<n>.json (n = argument index) and a one-line summary is printed.
n=0
for spec in "$@"; do
  envs="${spec%%::*}"; args=""
  [[ "$spec" == *"::"* ]] && args="${spec#*::}"
  env $envs timeout 300 python bench.py --no-cpu-baseline --no-e2e $args > "gpurun_out/ab_$n.json" 2>/dev/null
  python - "$n" "$spec" <<'PY'
import json, sys
n, spec = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/ab_{n}.json")); r = d["roofline"]
    print(f"[{n}] {spec:40s} {d['value']/1e12:.3f}e12  pass {d['ms_per_step']:.4f} ms  "
          f"steps {[round(v, 4) for v in d['step_p50_ms'].values()]}  k_stream {r['kernel_ms_mean']:.4f} ms  "
          f"frac {r['frac']:.3f}  surv {d['pruning']['survivors']}")
except Exception as e:
    print(f"[{n}] {spec}: failed ({e})")
PY
  n=$((n+1))
done
