"""C-ABI boundary features on the GPU: the xgr_config allocator hooks and the host-logits
step (xgr_beam_step_host). Both must give results identical to the default path (same kernels, same
inputs), and the search itself is checked against the oracle on every step."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

V, ND, BW, B = 1024, 2, 64, 2   # step 2 is a dense step (600 children per level-1 node)


def _items():
    from synth import make_items
    return make_items(600 * 1024, V, ND, 99)


def _logits():
    from synth import make_logits
    return [make_logits((B, 1 if t == 0 else BW, V), 4321 + t, 2.0) for t in range(ND)]


def _run(bs, xs, where, host=False, pin=True):
    """Steps the search, checks every step against the oracle, returns the host outputs."""
    import torch

    from oracle import xbeam_oracle as O
    from tests.parity import compare_step
    voc = O.Vocabulary(_items(), V, ND)
    states = [O.BeamState.root() for _ in range(B)]
    hp, ht = [], []
    for t, x in enumerate(xs):
        xt = torch.from_numpy(x)
        if host:
            xt = xt.pin_memory() if pin else xt
        else:
            xt = xt.cuda()
        bs.step(xt)
        v = bs.view()
        par, tok = v["parent"].cpu().numpy(), v["token"].cpu().numpy()
        sc, nl = v["score"].cpu().numpy(), v["n_live"].cpu().numpy()
        for r in range(B):
            compare_step(voc, states[r], x[r], BW, par[r], tok[r], sc[r], nl[r], where=f"{where} r{r} t{t + 1}")
        hp.append(par.copy())
        ht.append(tok.copy())
        states = [O.state_from_history([h[r] for h in hp], [h[r] for h in ht], sc[r], nl[r]) for r in range(B)]
    return bs.finalize(on_device=False)


def _same(a, b):
    for k in ("tokens", "item_rank", "score", "n_live"):
        np.testing.assert_array_equal(np.asarray(a[k]), np.asarray(b[k]), err_msg=k)


def test_torch_allocator_hooks_same_results():
    import torch

    import paper_2512_11529_b200 as xgr
    xs = _logits()
    ref = xgr.BeamSearch(V, ND, BW, B, device=0)
    ref.mask_build(_items())
    out_ref = _run(ref, xs, "default alloc")
    ref.close()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated(0)
    bs = xgr.BeamSearch(V, ND, BW, B, device=0, allocator="torch")
    bs.mask_build(_items())
    assert bs.alloc_calls[0] > 20   # the workspace and the trie came from the hooks
    assert torch.cuda.memory_allocated(0) > before   # ... i.e. from torch's caching allocator
    out = _run(bs, xs, "torch alloc")
    _same(out_ref, out)
    bs.close()
    assert bs.alloc_calls[0] == bs.alloc_calls[1]   # everything handed back
    assert torch.cuda.memory_allocated(0) == before


@pytest.mark.parametrize("pin", [True, False])
def test_host_logits_step_same_results(pin):
    import paper_2512_11529_b200 as xgr
    xs = _logits()
    ref = xgr.BeamSearch(V, ND, BW, B, device=0)
    ref.mask_build(_items())
    out_ref = _run(ref, xs, "device logits")
    ref.close()
    bs = xgr.BeamSearch(V, ND, BW, B, device=0)
    bs.mask_build(_items())
    for rep in range(2):   # the second search reuses the staging buffer
        out = _run(bs, xs, f"host logits (pinned {pin}, search {rep})", host=True, pin=pin)
        _same(out_ref, out)
    bs.close()


def test_host_step_bf16_and_errors():
    import ctypes

    import torch

    import paper_2512_11529_b200 as xgr
    from paper_2512_11529_b200 import binding
    bs = xgr.BeamSearch(V, ND, BW, B, device=0)
    bs.mask_build(_items())
    x = torch.randn(B, 1, V).to(torch.bfloat16).pin_memory()
    bs.step(x)   # bf16 host logits: the root step (sparse route) accepts them
    with pytest.raises(binding.XgrError) as e:   # ld < V
        binding.xgr_beam_step_host(bs.ctx, B, ctypes.c_void_p(x.data_ptr()), 0, BW, V - 1, None)
    assert e.value.name == "XGR_ERR_INVALID_ARG"
    with pytest.raises(binding.XgrError) as e:   # unknown dtype
        binding.xgr_beam_step_host(bs.ctx, B, ctypes.c_void_p(x.data_ptr()), 7, BW, V, None)
    assert e.value.name == "XGR_ERR_UNSUPPORTED"
    bs.close()


def test_host_logits_c2_full_size_bitwise():
    """C2 at full size (dense steps over 8192 rows) through xgr_beam_step_host from pinned memory:
    bitwise the device-logits path's states and outputs."""
    import torch

    import paper_2512_11529_b200 as xgr
    from synth import config, make_items, make_logits_torch
    c = config("C2")
    items = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    Bc, bw, Vc = c["batch"], c["beam_width"], c["vocab"]
    steps = [make_logits_torch((Bc, 1 if t == 0 else bw, Vc), 11 * t + 1, 2.0) for t in range(c["nd"])]
    res = []
    for host in (False, True):
        bs = xgr.BeamSearch(Vc, c["nd"], bw, Bc)
        bs.mask_build(items)
        per = []
        for lg in steps:
            bs.step(lg.cpu().pin_memory() if host else lg)
            v = bs.view()
            per.append({k: v[k].cpu().numpy().copy() for k in ("parent", "token", "score", "n_live")})
        res.append((bs.finalize(on_device=False), per))
        bs.close()
    _same(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        for k in a:
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    torch.cuda.synchronize()
