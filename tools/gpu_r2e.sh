#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab.sh "XGR_SEED_KERNEL=2 XGR_DEBUG_FLAGS=4194304::--steps 20" "XGR_SEED_KERNEL=0 XGR_DEBUG_FLAGS=4194304::--steps 20" "XGR_SEED_KERNEL=0::--steps 20" "XGR_SEED_KERNEL=2::--steps 20" "XGR_SEED_KERNEL=0::--steps 20 --logits bf16" "XGR_SEED_KERNEL=2::--steps 20 --logits bf16" "XGR_SEED_KERNEL=0::--steps 20 --config C2" "XGR_SEED_KERNEL=2::--steps 20 --config C2" "XGR_SEED_KERNEL=0::--steps 20 --sigma 4" > gpurun_out/ab_seed.txt 2>&1
cat gpurun_out/ab_seed.txt
timeout 2400 python -m pytest tests -q -m gpu -x -k "c2_full or c3_full or c3_sigma4 or pruning or bf16 or topk or graph or random_tries or skewed or c1" > gpurun_out/gputests_e.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_e.log
