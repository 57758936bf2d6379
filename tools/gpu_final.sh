#!/bin/bash
# Round-end measurement on one B200: bench lines of every config, the default bench exactly as the
# driver runs it, the reference arm, the ncu launch list of the default bench and one ncu --set full
# capture of the dominant kernel per config (profiles/ncu_k_stream_*_traffic.json via
# tools/traffic_json.py, read back on the dev box). Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/final_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final_smi.txt 2>&1
run() { n=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final_$n.json 2> gpurun_out/final_$n.err; echo "bench $n rc=$?"; }
run default
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "reference rc=$?"
run C3s4 --sigma 4 --no-cpu-baseline --no-e2e
run C3bf16 --logits bf16 --no-cpu-baseline --no-e2e
run C2 --config C2 --no-cpu-baseline --no-e2e
timeout 1500 python bench.py --config C3Z --no-cpu-baseline --no-e2e > gpurun_out/final_C3Z.json 2> gpurun_out/final_C3Z.err; echo "bench C3Z rc=$?"
run C4 --config C4 --steps 10 --no-cpu-baseline
run C5w --config C5 --split weak --steps 10 --no-cpu-baseline --no-e2e
run C3Zb --config C3Z --no-cpu-baseline --no-e2e --steps 10
run C5 --config C5 --steps 10 --no-cpu-baseline
run heap --paper-heap --no-graph --steps 10 --no-cpu-baseline --no-e2e
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --profile --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final_launches.log 2>&1; echo "launch list rc=$?"
R1='(\(int\))?'
KEEP_REP=1 bash tools/ncu_traffic.sh C3_f32 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0, float, ${R1}256, ${R1}1" C3 f32 2 -
bash tools/ncu_traffic.sh C3_f32_s4 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0, float, ${R1}256, ${R1}1" C3 f32 4 - --sigma 4
bash tools/ncu_traffic.sh C3_bf16 "k_stream<${R1}32, ${R1}1, ${R1}4, ${R1}3, ${R1}0, __nv_bfloat16, ${R1}256, ${R1}1" C3 bf16 2 - --logits bf16
bash tools/ncu_traffic.sh C2_f32 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0, float, ${R1}256, ${R1}1" C2 f32 2 - --config C2
bash tools/ncu_traffic.sh C4_f32 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}0, float, ${R1}256, ${R1}2" C4 f32 2 - --config C4
bash tools/ncu_traffic.sh C5w_f32 "k_stream2<${R1}3>" C5 f32 2 weak --config C5 --split weak
# the shard line's stats pass: skip the 8 root-step launches of the warm-up pass (one per local shard)
LSKIP=8 bash tools/ncu_traffic.sh C5s_f32 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}1, float, ${R1}256, ${R1}1" C5 f32 2 - --config C5
# the shard bench line again, now reading the capture just taken
cp gpurun_out/final/profiles/ncu_k_stream_C5_f32_traffic.json profiles/ && run C5 --config C5 --steps 10 --no-cpu-baseline
python tools/launch_shares.py gpurun_out/final_launches.csv > gpurun_out/final/r02_launches_xgr.txt 2>&1
rm -f gpurun_out/final_launches.csv.gz
du -sh gpurun_out
