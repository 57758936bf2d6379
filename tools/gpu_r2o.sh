#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
rm -rf gpurun_out/final/profiles
R1='(\(int\))?'
bash tools/ncu_traffic.sh C5w_f32 "k_stream2<${R1}3>" C5 f32 2 weak --config C5 --split weak
bash tools/ncu_traffic.sh C5s_f32 "k_stream<${R1}32, ${R1}1, ${R1}2, ${R1}3, ${R1}1, float, ${R1}256, ${R1}1" C5 f32 2 - --config C5
bash tools/ab.sh "XGR_SEED_KERNEL=3::--steps 20" "::--steps 20" "XGR_SEED_KERNEL=3::--steps 20 --config C2" "::--steps 20 --config C2" "XGR_THETA_ROWS=4::--steps 20" "XGR_THETA_ROWS=12::--steps 20" > gpurun_out/ab_o.txt 2>&1
cat gpurun_out/ab_o.txt
XGR_SEED_KERNEL=3 timeout 1200 python -m pytest tests -q -m gpu -x -k "random_tries or c2_full or skewed or pruning" > gpurun_out/gputests_o.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_o.log
