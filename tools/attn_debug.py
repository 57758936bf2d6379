"""Development check: where the staged-attention output departs from the oracle (rows/cols)."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11529_b200 as xgr
from oracle import attention as A
from synth import make_attn_inputs
for shape in [(1, 4, 4, 2, 70, 3, 2), (1, 4, 4, 2, 70, 3, 0), (1, 4, 4, 2, 64, 3, 2), (1, 4, 4, 2, 130, 3, 2), (1, 64, 8, 2, 300, 3, 2), (1, 64, 8, 2, 300, 3, 0)]:
    n_req, bw, hq, hkv, ls, nd, n = shape
    q, ks, vs, ku, vu = make_attn_inputs(n_req, bw, hq, hkv, 128, ls, nd, seed=1)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()
    out = xgr.attn_staged(bf(q), bf(ks), bf(vs), bf(ku), bf(vu), n, hkv, 1 / math.sqrt(128)).float().cpu().numpy()
    ref, _ = A.staged_attention(q[0], ks[0], vs[0], ku[0], vu[0], n, 1 / math.sqrt(128))
    err = np.abs(out[0] - ref)
    bad = ~(err < 0.02)
    print(shape, "bad frac", bad.mean(), "nan frac", np.isnan(out).mean(), "bad beams", np.unique(np.nonzero(bad)[0])[:10],
          "bad cols", np.unique(np.nonzero(bad)[2])[:20], "max err", np.nanmax(err))
