"""GPU parity of the staged shared/unshared attention (second workload;
PAPER.md L339) against the fp64 oracle (oracle/attention.py), through the
C ABI (xgr_attn_staged / xgr_attn_shared / xgr_attn_unshared / xgr_attn_merge).

Tolerance (reading A3): q, k, v are bf16 (exact on both sides); S = Q K^T is accumulated
in fp32 (error ~ d * 2^-24 relative); the softmax weights p <= 2^8 are rounded to bf16 for the
P V product (relative 2^-9 each), so the shared stage's normalised output is within
2^-8 * sum_j p_j |v_j| / sum_j p_j of the exact value (factor 2 of slack), plus the bf16 rounding
of the output itself (2^-8 relative). m, s and lse see only fp32 rounding and ex2.approx
(2^-22 relative): 1e-5.
"""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from synth import ATTN_CONFIGS, make_attn_inputs

pytestmark = pytest.mark.gpu


def _bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


def _bound(q, ks, vs, ku, vu, n, scale, ref):
    """2^-7 * (sum p |v| / sum p) + 2^-8 |ref|: the P-rounding and output-rounding bound."""
    wabs, _ = A.full_attention(q, ks, np.abs(vs), ku, np.abs(vu), n, scale)
    return 2.0 ** -7 * wabs + 2.0 ** -8 * np.abs(ref) + 1e-6


def _run_staged(xgr, q, ks, vs, ku, vu, n, hkv, scale):
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    out = xgr.attn_staged(_bf(q), _bf(ks) if ks.shape[1] else None, _bf(vs) if ks.shape[1] else None,
                          _bf(ku), _bf(vu), n, hkv, scale, lse=lse)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy()


SHAPES = [  # (n_req, bw, hq, hkv, ls, nd, n)
    (2, 4, 4, 2, 70, 3, 2),        # A1-like: one ragged M tile, two key tiles with a ragged tail
    (1, 40, 8, 2, 64, 3, 3),       # G = 4: 160 rows = two M tiles (ragged), exactly one key tile
    (2, 16, 8, 8, 1, 3, 1),        # G = 1, one prompt token
    (1, 8, 16, 1, 130, 2, 0),      # G = 16, no unshared tokens, 3 key tiles
    (1, 3, 2, 1, 65, 3, 3),        # tiny bw, ragged by one key
    (1, 64, 8, 2, 300, 3, 1),      # 256 rows = two full M tiles, 5 key tiles
    (1, 2, 128, 1, 50, 3, 2),      # G = 128: one beam per tile
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("sigma_q", [1.0, 4.0])
def test_staged_matches_oracle(shape, sigma_q):
    import paper_2512_11529_b200 as xgr
    n_req, bw, hq, hkv, ls, nd, n = shape
    d = 128
    scale = 1.0 / math.sqrt(d)
    q, ks, vs, ku, vu = make_attn_inputs(n_req, bw, hq, hkv, d, ls, nd, seed=hash(shape) & 0xFFFF, sigma_q=sigma_q)
    out, lse = _run_staged(xgr, q, ks, vs, ku, vu, n, hkv, scale)
    for r in range(n_req):
        ref, rlse = A.staged_attention(q[r], ks[r], vs[r], ku[r], vu[r], n, scale)
        bnd = _bound(q[r], ks[r], vs[r], ku[r], vu[r], n, scale, ref)
        err = np.abs(out[r] - ref)
        assert np.all(err <= bnd), f"r{r}: max err {err.max()} (bound there {bnd.flat[err.argmax()]})"
        assert np.allclose(lse[r], rlse, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("trial", range(12))
def test_random_shapes(trial):
    """Random shapes (prompt 0-400 tokens, 1-70 beams, G = 1-8, 1-4 KV heads, 0-3 own tokens)
    through both epilogue paths (staged or per-thread unshared rows, depending on the shape)."""
    import paper_2512_11529_b200 as xgr
    rng = np.random.default_rng(9000 + trial)
    G = int(rng.choice([1, 2, 4, 8])); hkv = int(rng.choice([1, 2, 4]))
    bw = int(rng.integers(1, 71)); ls = int(rng.integers(0, 401)); nd = 3
    n = int(rng.integers(0 if ls > 0 else 1, 4))
    n_req = int(rng.integers(1, 3))
    scale = 1.0 / math.sqrt(128)
    q, ks, vs, ku, vu = make_attn_inputs(n_req, bw, G * hkv, hkv, 128, ls, nd, seed=trial,
                                         sigma_q=float(rng.choice([1.0, 3.0])))
    out, lse = _run_staged(xgr, q, ks, vs, ku, vu, n, hkv, scale)
    for r in range(n_req):
        ref, rlse = A.staged_attention(q[r], ks[r], vs[r], ku[r], vu[r], n, scale)
        bnd = _bound(q[r], ks[r], vs[r], ku[r], vu[r], n, scale, ref)
        assert np.all(np.abs(out[r] - ref) <= bnd), (trial, G, hkv, bw, ls, n)
        assert np.allclose(lse[r], rlse, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_empty_prompt_unshared_only(n):
    """ls = 0: the shared stage is the empty partial; output = unshared attention."""
    import paper_2512_11529_b200 as xgr
    q, ks, vs, ku, vu = make_attn_inputs(2, 6, 4, 2, 128, 0, 3, seed=40 + n)
    out, lse = _run_staged(xgr, q, ks, vs, ku, vu, n, 2, 0.1)
    for r in range(2):
        ref, rlse = A.staged_attention(q[r], ks[r], vs[r], ku[r], vu[r], n, 0.1)
        assert np.allclose(out[r], ref, rtol=2 ** -7, atol=1e-6)
        assert np.allclose(lse[r], rlse, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("shape", [(2, 4, 4, 2, 70), (1, 40, 8, 2, 129), (1, 5, 4, 4, 0), (1, 8, 16, 2, 1)])
def test_shared_partials(shape):
    """xgr_attn_shared returns the canonical partial (m = true max, s, o) of S:L136-139."""
    import paper_2512_11529_b200 as xgr
    n_req, bw, hq, hkv, ls = shape
    scale = 1.0 / math.sqrt(128)
    q, ks, vs, _, _ = make_attn_inputs(n_req, bw, hq, hkv, 128, ls, 1, seed=7 + ls, sigma_q=2.0)
    m, s, o = xgr.attn_shared(_bf(q), _bf(ks) if ls else None, _bf(vs) if ls else None, hkv, scale)
    torch.cuda.synchronize()
    m, s, o = m.cpu().numpy(), s.cpu().numpy(), o.cpu().numpy()
    for r in range(n_req):
        rm, rs, ro = A.attend_shared(q[r], ks[r], vs[r], scale)
        if ls == 0:
            assert np.all(np.isneginf(m[r])) and np.all(s[r] == 0) and np.all(o[r] == 0)
            continue
        assert np.allclose(m[r], rm, rtol=1e-5, atol=1e-6)
        assert np.allclose(s[r], rs, rtol=1e-5)
        norm, rnorm = o[r] / s[r][..., None], ro / rs[..., None]
        _, _, rabs = A.attend_shared(q[r], ks[r], np.abs(vs[r]), scale)
        assert np.all(np.abs(norm - rnorm) <= 2.0 ** -7 * rabs / rs[..., None] + 1e-6)


def test_unshared_partials_and_merge():
    """xgr_attn_unshared and xgr_attn_merge vs the oracle, including a
    merge with an empty partial (identity)."""
    import paper_2512_11529_b200 as xgr
    scale = 0.09
    q, ks, vs, ku, vu = make_attn_inputs(2, 6, 8, 2, 128, 37, 3, seed=11)
    for n in range(0, 4):
        m, s, o = xgr.attn_unshared(_bf(q), _bf(ku), _bf(vu), n, 2, scale)
        torch.cuda.synchronize()
        for r in range(2):
            rm, rs, ro = A.attend_unshared(q[r], ku[r], vu[r], n, scale)
            if n == 0:
                assert np.all(np.isneginf(m[r].cpu().numpy())) and np.all(s[r].cpu().numpy() == 0)
                continue
            assert np.allclose(m[r].cpu().numpy(), rm, rtol=1e-5, atol=1e-6)
            assert np.allclose(s[r].cpu().numpy(), rs, rtol=1e-5)
            assert np.allclose(o[r].cpu().numpy(), ro, rtol=1e-4, atol=1e-5)
    # merge of float partials given exactly (fp32 values) on both sides
    rng = np.random.default_rng(5)
    rows = 300
    m1 = rng.standard_normal(rows).astype(np.float32); s1 = (1 + rng.random(rows)).astype(np.float32)
    o1 = rng.standard_normal((rows, 128)).astype(np.float32)
    m2 = rng.standard_normal(rows).astype(np.float32) * 3; s2 = (1 + rng.random(rows)).astype(np.float32)
    o2 = rng.standard_normal((rows, 128)).astype(np.float32)
    m2[:20] = -np.inf; s2[:20] = 0; o2[:20] = 0          # empty second partial
    m1[20:30] = -np.inf; s1[20:30] = 0; o1[20:30] = 0    # empty first partial
    T = lambda x: torch.from_numpy(x).cuda()
    out, lse = xgr.attn_merge((T(m1), T(s1), T(o1)), (T(m2), T(s2), T(o2)), with_lse=True)
    ref, rlse = A.merge_partials((m1.astype(np.float64), s1.astype(np.float64), o1.astype(np.float64)),
                                 (m2.astype(np.float64), s2.astype(np.float64), o2.astype(np.float64)))
    assert np.allclose(out.cpu().numpy(), ref, rtol=1e-5, atol=1e-6)
    assert np.allclose(lse.cpu().numpy(), rlse, rtol=1e-6, atol=1e-6)


def test_deterministic_and_beam_isolation():
    import paper_2512_11529_b200 as xgr
    q, ks, vs, ku, vu = make_attn_inputs(1, 32, 8, 2, 128, 200, 3, seed=3)
    a, _ = _run_staged(xgr, q, ks, vs, ku, vu, 3, 2, 0.088)
    b, _ = _run_staged(xgr, q, ks, vs, ku, vu, 3, 2, 0.088)
    assert np.array_equal(a, b)
    ku2 = ku.copy(); ku2[0, 5] = -ku2[0, 5]
    c, _ = _run_staged(xgr, q, ks, vs, ku2, vu, 3, 2, 0.088)
    others = [i for i in range(32) if i != 5]
    assert np.array_equal(a[0, others], c[0, others]) and not np.array_equal(a[0, 5], c[0, 5])


def test_bw512_long_prompt_sampled():
    """A3 (BW 512, prompt 3072: the paper's largest beam width and input length, PAPER.md
    L559-566), sampled beams of every request against the oracle."""
    import paper_2512_11529_b200 as xgr
    c = ATTN_CONFIGS["A3"]
    n_req, bw, hq, hkv, d, ls, nd = (c[k] for k in ("n_req", "bw", "hq", "hkv", "d", "ls", "nd"))
    scale = 1.0 / math.sqrt(d)
    q, ks, vs, ku, vu = make_attn_inputs(n_req, bw, hq, hkv, d, ls, nd, seed=77, sigma_q=2.0)
    out, lse = _run_staged(xgr, q, ks, vs, ku, vu, 2, hkv, scale)
    rng = np.random.default_rng(1)
    for r in range(n_req):
        beams = np.sort(rng.choice(bw, 4, replace=False))
        ref, rlse = A.staged_attention(q[r][beams], ks[r], vs[r], ku[r][beams], vu[r][beams], 2, scale)
        bnd = _bound(q[r][beams], ks[r], vs[r], ku[r][beams], vu[r][beams], 2, scale, ref)
        assert np.all(np.abs(out[r][beams] - ref) <= bnd)
        assert np.allclose(lse[r][beams], rlse, rtol=1e-5, atol=1e-5)


def test_full_size_sampled():
    """A2 (bench workload: 16 requests x BW 256 x 32 heads, 8 KV heads, prompt 1024, step 3 with
    3 own tokens per beam) in the launch configuration the bench times; the oracle checks sampled
    beams of sampled requests (beams are independent, so a beam subset is an exact sub-problem)."""
    import paper_2512_11529_b200 as xgr
    c = ATTN_CONFIGS["A2"]
    n_req, bw, hq, hkv, d, ls, nd = (c[k] for k in ("n_req", "bw", "hq", "hkv", "d", "ls", "nd"))
    scale = 1.0 / math.sqrt(d)
    q, ks, vs, ku, vu = make_attn_inputs(n_req, bw, hq, hkv, d, ls, nd, seed=2025)
    out, lse = _run_staged(xgr, q, ks, vs, ku, vu, nd, hkv, scale)
    rng = np.random.default_rng(0)
    for r in (0, 7, n_req - 1):
        beams = np.sort(rng.choice(bw, 6, replace=False))
        beams[-1] = bw - 1
        ref, rlse = A.staged_attention(q[r][beams], ks[r], vs[r], ku[r][beams], vu[r][beams], nd, scale)
        bnd = _bound(q[r][beams], ks[r], vs[r], ku[r][beams], vu[r][beams], nd, scale, ref)
        assert np.all(np.abs(out[r][beams] - ref) <= bnd)
        assert np.allclose(lse[r][beams], rlse, rtol=1e-5, atol=1e-5)
