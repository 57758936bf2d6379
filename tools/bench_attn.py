"""Measure the staged shared/unshared attention (second workload) on the A2
workload (synth.ATTN_CONFIGS: Qwen3-4B attention layer -- 32 query heads, 8 KV heads, d 128 --
16 requests x BW 256 beams, prompt 1024, decode step 3 with 3 own tokens per beam).

Prints one JSON line: xgr_attn_staged time (CUDA events on the launch stream, L2 flushed by a
256 MiB write before every launch), algorithmic tensor FLOPs (QK^T + PV of every query row
against every prompt key: 4 * rows * ls * d) against the measured dense bf16 peak, the HBM bytes
the kernel must move at least (q, out, shared K/V once per request, unshared K/V of the beams),
and, for comparison, the library flash-attention (flash_attn 2, sm_80 code path) of the shared
stage with the beams as a query sequence, plus the bytes a per-beam (PagedAttention-like) kernel
would read."""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_11529_b200 as xgr  # noqa: E402
from synth import ATTN_CONFIGS  # noqa: E402


def timed(fn, iters, flush):
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


def main():
    cfg = os.environ.get("ATTN_CFG", "A2")
    c = ATTN_CONFIGS[cfg]
    n_req, bw, hq, hkv, d, ls, nd = (c[k] for k in ("n_req", "bw", "hq", "hkv", "d", "ls", "nd"))
    ls = int(os.environ.get("ATTN_LS", ls))
    nu = int(os.environ.get("ATTN_NU", nd))
    scale = 1.0 / math.sqrt(d)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    rnd = lambda *s: torch.randn(s, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    q = rnd(n_req, bw, hq, d)
    ks, vs = rnd(n_req, ls, hkv, d), rnd(n_req, ls, hkv, d)
    ku, vu = rnd(n_req, bw, nd, hkv, d), rnd(n_req, bw, nd, hkv, d)
    out = torch.empty_like(q)
    run = lambda: xgr.attn_staged(q, ks, vs, ku, vu, nu, hkv, scale, out=out)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    iters = int(os.environ.get("ATTN_ITERS", "20"))
    ts = timed(run, iters, flush)
    ms = sorted(ts)[len(ts) // 2]
    ms_mean = sum(ts) / len(ts)
    rows = n_req * bw * hq
    flops = 4.0 * rows * ls * d
    byts = (q.numel() + out.numel() + ks.numel() + vs.numel() + n_req * bw * nu * hkv * d * 2) * 2
    per_beam_bytes = (q.numel() + out.numel()) * 2 + n_req * bw * (ls + nd) * hkv * d * 2 * 2
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_tf, peak_bw = peaks["bf16_tflops"], peaks["hbm_gbs"]
        src = "measured (MEASURED_PEAKS.json bf16_tflops, hbm_gbs)"
    except (OSError, KeyError):
        peak_tf, peak_bw, src = 2250.0, 7672.0, "nominal"
    tf = flops / (ms_mean / 1e3) / 1e12
    res = {"kernel": "k_attn_shared<false> (tcgen05 shared stage + fused unshared stage and merge)",
           "workload": cfg, "n_req": n_req, "bw": bw, "hq": hq, "hkv": hkv, "d": d, "ls": ls,
           "n_unshared": nu, "ms_mean": ms_mean, "ms_p50": ms, "ms_all": ts,
           "roofline": {"bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
                        "frac": tf / peak_tf, "peak_source": src, "alg_flops": flops},
           "hbm": {"alg_bytes": byts, "achieved_gbs": byts / (ms_mean / 1e3) / 1e9, "peak_gbs": peak_bw,
                   "per_beam_kernel_bytes": per_beam_bytes},
           "l2": "flushed (256 MiB write) before every launch"}
    try:
        from flash_attn import flash_attn_func
        fa = lambda: flash_attn_func(q, ks, vs, softmax_scale=scale, causal=False)
        for _ in range(3):
            fa()
        tfa = timed(fa, iters, flush)
        res["flash_attn2_shared_stage_ms_mean"] = sum(tfa) / len(tfa)
        res["flash_attn2_tflops"] = flops / (sum(tfa) / len(tfa) / 1e3) / 1e12
    except Exception as e:  # library comparison only
        res["flash_attn2_shared_stage_ms_mean"] = f"unavailable: {type(e).__name__}: {e}"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
