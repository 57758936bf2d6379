"""Development check: one small dense-route beam search (V 8192, BW 64, ND 3, 4 requests) in the
fused seed + step mode (XGR_SEED_KERNEL=4) for compute-sanitizer runs, checked against the
default seed mode bitwise (same kernels otherwise)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11529_b200 as xgr  # noqa: E402
from synth import make_items, make_logits_torch  # noqa: E402

V, ND, BW, B = 8192, 3, 64, 4
items = make_items(2_000_000, V, ND, 777)
steps = [make_logits_torch((B, 1 if t == 0 else BW, V), 90 + t, 2.0) for t in range(ND)]
outs = []
for mode in ("4", "1"):
    os.environ["XGR_SEED_KERNEL"] = mode
    bs = xgr.BeamSearch(V, ND, BW, B, flags=2 | 4)   # counters, every step on the dense route
    bs.mask_build(items)
    for lg in steps:
        bs.step(lg)
    outs.append(bs.finalize(on_device=False))
    print("mode", mode, "counters", bs.counters())
    bs.close()
for k in ("tokens", "item_rank", "score", "n_live"):
    np.testing.assert_array_equal(outs[0][k], outs[1][k], err_msg=k)
print("fused == default: ok")
