"""xgr_kv_reorder against the gather oracle (oracle/kv_reorder.py, pinned by
SPEC's examples in tests/test_kv_oracle.py): bit-exact bytes, in place, any map (including the
non-monotone ones that defeat SPEC's two-pass scheme), dead slots untouched."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import kv_reorder as K  # noqa: E402


@pytest.fixture(scope="module")
def xgr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11529_b200 as xgr
    return xgr


def _expected(cache_np, src_np):
    out = cache_np.copy()
    n_req, n_panel, bw, _ = cache_np.shape
    for r in range(n_req):
        s = src_np[r, :bw].astype(np.int64)
        live = s >= 0
        for p in range(n_panel):
            g = K.gather(cache_np[r, p], np.where(live, s, np.arange(bw)))
            out[r, p] = g
    return out


def test_spec_examples_bytes(xgr):
    rows = np.array([[ord(c)] * 16 for c in "ABCD"], np.uint8)[None, None]   # [1][1][4][16]
    for src, want in (([1, 2, 2, 3], "BCCD"), ([0, 0, 1, 2], "AABC"), ([0, 1, 2, 3], "ABCD"),
                      ([3, 2, 1, 0], "DCBA"), ([2, 0, 1, 0], "CABA")):
        c = torch.from_numpy(rows.copy()).cuda()
        xgr.kv_reorder(c, torch.tensor([src], dtype=torch.int32, device="cuda"))
        got = "".join(chr(v) for v in c[0, 0, :, 0].cpu().tolist())
        assert got == want, (src, got)
        assert torch.all(c[0, 0] == c[0, 0, :, :1])   # whole rows moved


@pytest.mark.parametrize("bw,row_elems,dtype", [(1, 8, torch.float16), (4, 24, torch.float16),
                                                (128, 520, torch.bfloat16), (256, 64, torch.float32),
                                                (512, 1032, torch.float16), (1024, 72, torch.int32)])
def test_random_maps_match_gather(xgr, bw, row_elems, dtype):
    rng = np.random.default_rng(bw + row_elems)
    n_req, n_panel = 3, 2
    es = torch.tensor([], dtype=dtype).element_size()
    pad = 16 // es                                             # padded beam stride (16 bytes)
    raw = torch.from_numpy(rng.integers(0, 256, size=(n_req, n_panel, bw, (row_elems + pad) * es),
                                        dtype=np.uint8))
    full = raw.cuda()
    cache = full.view(dtype)[..., :row_elems]                 # strided view: beam stride > row
    src = rng.integers(-1, bw, size=(n_req, bw + 5)).astype(np.int32)   # -1: dead slot; ld > bw
    src[0, :bw] = np.arange(bw)[::-1]                         # a reversal (non-monotone swaps)
    xgr.kv_reorder(cache, torch.from_numpy(src).cuda())
    got = full.cpu().numpy()
    rb = row_elems * es
    want = _expected(raw.numpy()[..., :rb], src)
    assert np.array_equal(got[..., :rb], want)
    assert np.array_equal(got[..., rb:], raw.numpy()[..., rb:])   # padding untouched


def test_after_a_beam_step(xgr):
    """The consumer the row is for: reorder a per-beam cache by the step's parent[]."""
    from synth import make_items, make_logits
    rng = np.random.default_rng(2)
    vocab, nd, bw, batch = 1024, 3, 64, 3
    items = make_items(20000, vocab, nd, 77)
    bs = xgr.BeamSearch(vocab, nd, bw, batch)
    bs.mask_build(items)
    cache = torch.from_numpy(rng.integers(0, 255, size=(batch, 4, bw, 256), dtype=np.uint8)).cuda()
    for t in range(nd):
        x = torch.from_numpy(make_logits((batch, 1 if t == 0 else bw, vocab), 40 + t, 2.0)).cuda()
        bs.step(x)
        par = bs.view()["parent"]
        before = cache.cpu().numpy()
        xgr.kv_reorder(cache, par)
        assert np.array_equal(cache.cpu().numpy(), _expected(before, par.cpu().numpy()))
    bs.finalize(on_device=True)


def test_argument_errors(xgr):
    c = torch.zeros((1, 1, 4, 16), dtype=torch.uint8, device="cuda")
    src = torch.zeros((1, 4), dtype=torch.int32, device="cuda")
    L = xgr.lib
    import ctypes
    vp = ctypes.c_void_p
    assert L.xgr_kv_reorder(vp(c.data_ptr()), 1, 1, 4, 16, 16, 64, 64, vp(src.data_ptr()), 4, None) == 0
    assert L.xgr_kv_reorder(vp(c.data_ptr()), 1, 1, 4, 12, 16, 64, 64, vp(src.data_ptr()), 4, None) != 0   # 16 B
    assert L.xgr_kv_reorder(vp(c.data_ptr()), 1, 1, 2000, 16, 16, 64, 64, vp(src.data_ptr()), 2000, None) != 0
    assert L.xgr_kv_reorder(vp(c.data_ptr()), 1, 1, 4, 32, 16, 64, 64, vp(src.data_ptr()), 4, None) != 0   # overlap
    assert L.xgr_kv_reorder(None, 1, 1, 4, 16, 16, 64, 64, vp(src.data_ptr()), 4, None) != 0
    assert L.xgr_kv_reorder(None, 0, 1, 4, 16, 16, 64, 64, None, 4, None) == 0   # empty: no-op
