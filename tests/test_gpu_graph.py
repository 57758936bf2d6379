"""A whole beam-search pass (ND steps + finalize) captured in one CUDA graph and replayed on new
logits gives bitwise the same result as eager execution (xSchedule "captures a
series of device-side operations ... in the form of a graph and submits them all at once";
include/xgr_beam.h: xgr_beam_step only enqueues, no sync, no allocation)."""
import numpy as np
import pytest
import torch

from synth import make_items, make_logits_torch

pytestmark = pytest.mark.gpu


def _outputs(bs):
    v = bs.outputs_view()
    return {k: t.clone() for k, t in v.items()}


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_graph_replay_matches_eager(dtype):
    import paper_2512_11529_b200 as xgr
    V, ND, BW, B = 8192, 3, 128, 8
    items = make_items(2_000_000, V, ND, 4242)
    bs = xgr.BeamSearch(V, ND, BW, B)
    bs.mask_build(items)
    rows = [1, BW, BW]
    logits = [torch.empty((B, rows[t], V), dtype=dtype, device="cuda") for t in range(ND)]

    def fill(seed):
        for t in range(ND):
            logits[t].copy_(make_logits_torch((B, rows[t], V), seed + t, 2.0).to(dtype))

    def one_pass():
        for t in range(ND):
            bs.step(logits[t])
        bs.finalize_in_place()

    fill(100)
    one_pass()                       # eager warm-up (also exercises every route once)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        one_pass()
    for seed in (200, 300):
        fill(seed)
        one_pass()                   # eager reference
        torch.cuda.synchronize()
        ref = _outputs(bs)
        fill(seed)
        g.replay()
        torch.cuda.synchronize()
        got = _outputs(bs)
        for k in ref:
            assert torch.equal(ref[k], got[k]), k
        assert int(got["n_live"].min()) == BW
    bs.close()
