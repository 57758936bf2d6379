"""Development check: one small V = 16384 beam search (C4-shaped: BW 512, ND 4) for
compute-sanitizer runs of the dense-route variants (XGR_SEED_MODE)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11529_b200 as xgr  # noqa: E402
from synth import make_items, make_logits_torch  # noqa: E402

V, ND, BW, B = 16384, 4, 512, int(os.environ.get("SAN_BATCH", "4"))
items = make_items(int(os.environ.get("SAN_ITEMS", "30000000")), V, ND, 4242)
bs = xgr.BeamSearch(V, ND, BW, B, flags=2)
bs.mask_build(items)
for t in range(ND):
    bs.step(make_logits_torch((B, 1 if t == 0 else BW, V), 50 + t, 2.0))
out = bs.finalize(on_device=False)
print("n_live", out["n_live"], "counters", bs.counters())
