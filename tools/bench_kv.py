"""Measure xgr_kv_reorder on a C3-shaped per-beam cache: BW = 256 beams per
request, one panel per (layer, K|V) of a 28-layer model with 8 KV heads x 128 dims in bf16 and
ND = 3 generated tokens (6 KiB per beam per panel), parents taken from real C3-like beam steps.
Prints one JSON line: algorithmic bytes (distinct source rows read + changed rows written) per
launch / mean CUDA-event time, against the measured HBM peak."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_11529_b200 as xgr  # noqa: E402
from synth import make_items, make_logits_torch  # noqa: E402


def main():
    B, BW, V, ND = int(os.environ.get("KV_BATCH", "32")), 256, 8192, 3
    layers, heads, dim = 28, 8, 128
    row_bytes = ND * heads * dim * 2
    n_panel = 2 * layers
    items = make_items(2_000_000, V, ND, 99)
    bs = xgr.BeamSearch(V, ND, BW, B)
    bs.mask_build(items)
    pars = []
    for t in range(ND):
        bs.step(make_logits_torch((B, 1 if t == 0 else BW, V), 900 + t, 2.0))
        pars.append(bs.view()["parent"].clone())
    bs.finalize(on_device=True)
    src = pars[-1]                                   # the last step's parents (a dense reshuffle)
    s = src.cpu().numpy()
    moved = reads = 0
    for r in range(B):
        ch = (s[r] >= 0) & (s[r] != np.arange(BW))
        moved += int(ch.sum())
        reads += len(set(s[r][ch].tolist()))
    alg = (moved + reads) * row_bytes * n_panel
    cache = torch.empty((B, n_panel, BW, row_bytes // 2), dtype=torch.bfloat16, device="cuda")
    cache.view(torch.int16).random_(-30000, 30000)
    for _ in range(3):
        xgr.kv_reorder(cache, src)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > L2 between launches
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        xgr.kv_reorder(cache, src)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except OSError:
        peak = 6650.0
    gbs = alg / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": "k_kv_reorder", "batch": B, "bw": BW, "panels": n_panel, "row_bytes": row_bytes,
                      "cache_bytes": B * n_panel * BW * row_bytes, "changed_rows_per_panel": moved,
                      "distinct_src_rows_per_panel": reads, "alg_bytes": alg, "ms_mean": ms,
                      "ms_all": ts, "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
                      "l2": "flushed (256 MiB write) before every launch"}))


if __name__ == "__main__":
    main()
