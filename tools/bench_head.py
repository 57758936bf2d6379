"""LM-head fusion at the sparse step at the C3 shape: batch 256 x BW 256,
V = 8192, 100M-item trie; step 3 (about 1.9 legal tokens per row) driven by hidden states of
width d = 2048 (bf16) and a bf16 LM head [8192][2048].

  fused:   xgr_beam_step_head (k_head: legal-token dot products only, + the sparse-step kernel)
  unfused: logits = hidden @ head^T (cuBLAS bf16 GEMM, bf16 out) + xgr_beam_step_ex(bf16)

Prints one JSON line with the step-3 times (CUDA events, mean over repetitions) and the k_head
byte roofline (hidden read once from HBM + the distinct LM-head rows)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_11529_b200 as xgr  # noqa: E402
from synth import config, make_items, make_logits_torch  # noqa: E402


def main():
    c = config("C3")
    B, BW, V, ND, d = c["batch"], c["beam_width"], c["vocab"], c["nd"], int(os.environ.get("HEAD_D", "2048"))
    items = make_items(c["n_items"], V, ND, c["trie_key"])
    bs = xgr.BeamSearch(V, ND, BW, B)
    bs.mask_build(items)
    del items
    lg = [make_logits_torch((B, 1 if t == 0 else BW, V), 11 * t + 1, 2.0) for t in range(ND - 1)]
    g = torch.Generator(device="cuda").manual_seed(5)
    head = (torch.randn((V, d), device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    hid = torch.randn((B, BW, d), device="cuda", generator=g).to(torch.bfloat16)
    logits_buf = torch.empty((B, BW, V), device="cuda", dtype=torch.bfloat16)
    reps = 10

    def run(fused, ev):
        for t in range(ND - 1):
            bs.step(lg[t])
        assert bs.next_is_sparse()
        ev[0].record()
        if fused:
            bs.step_head(hid, head)
        else:
            torch.matmul(hid, head.T, out=logits_buf)
            bs.step(logits_buf)
        ev[1].record()
        bs.finalize_in_place()

    res = {}
    for fused in (True, False):
        ts = []
        for k in range(reps + 2):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            run(fused, ev)
            torch.cuda.synchronize()
            if k >= 2:
                ts.append(ev[0].elapsed_time(ev[1]))
        res["fused" if fused else "unfused"] = sum(ts) / len(ts)
    hbytes = B * BW * d * 2
    wbytes = V * d * 2
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except OSError:
        peak = 6650.0
    ach = (hbytes + wbytes) / (res["fused"] / 1e3) / 1e9
    print(json.dumps({"workload": "C3 step 3 (sparse), hidden d=%d bf16, head [%d][%d] bf16" % (d, V, d),
                      "fused_step_ms": res["fused"], "unfused_gemm_plus_step_ms": res["unfused"],
                      "speedup": res["unfused"] / res["fused"],
                      "fused_alg_bytes": hbytes + wbytes, "fused_achieved_gbs": ach, "peak_gbs": peak,
                      "fused_frac": ach / peak, "reps": reps,
                      "note": "fused time includes k_head and the sparse-step kernel; alg bytes = hidden once + head once"}))


if __name__ == "__main__":
    main()
