"""Pins for oracle/attention.py (staged shared/unshared attention), each fixed
by something other than the oracle: SPEC.md worked examples, closed forms, and an
independent library routine (torch's scaled_dot_product_attention in fp64 on the CPU, with the
beam's own-token visibility as an explicit mask)."""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from synth import make_attn_inputs


def sdpa_reference(q, ks, vs, ku, vu, n, scale):
    """torch SDPA over [prompt ; all beams' own tokens] with a mask exposing beam b's t < n only."""
    bw, hq, d = q.shape
    ls, hkv = ks.shape[0], ks.shape[1]
    G = hq // hkv
    nd = ku.shape[1]
    # keys: [hkv][ls + bw*nd][d]
    k = np.concatenate([ks.transpose(1, 0, 2), ku.transpose(2, 0, 1, 3).reshape(hkv, bw * nd, d)], axis=1)
    v = np.concatenate([vs.transpose(1, 0, 2), vu.transpose(2, 0, 1, 3).reshape(hkv, bw * nd, d)], axis=1)
    k = torch.from_numpy(np.repeat(k, G, axis=0)).double()     # query head h -> kv head h // G
    v = torch.from_numpy(np.repeat(v, G, axis=0)).double()
    qq = torch.from_numpy(q.transpose(1, 0, 2).copy()).double()  # [hq][bw][d]
    mask = torch.zeros(bw, ls + bw * nd, dtype=torch.bool)
    mask[:, :ls] = True
    for b in range(bw):
        mask[b, ls + b * nd: ls + b * nd + n] = True
    out = torch.nn.functional.scaled_dot_product_attention(qq, k, v, attn_mask=mask, scale=scale)
    return out.numpy().transpose(1, 0, 2)


def test_empty_prompt_is_empty_partial():
    q = np.ones((2, 2, 4)); ks = np.zeros((0, 1, 4))
    m, s, o = A.attend_shared(q, ks, ks, 0.5)
    assert np.all(np.isneginf(m)) and np.all(s == 0) and np.all(o == 0)


def test_single_key_weight_one():
    q = np.array([[[1.0, 0.0]]]); k = np.array([[[0.0, 3.0]]]); v = np.array([[[2.5, -1.0]]])
    m, s, o = A.attend_shared(q, k, v, 1.0)
    assert m[0, 0] == 0.0 and s[0, 0] == 1.0 and np.array_equal(o[0, 0], v[0, 0])
    ku = k[None]; vu = v[None]                        # [bw=1][nd=1][hkv=1][d]
    m, s, o = A.attend_unshared(q, ku, vu, 1, 1.0)
    assert s[0, 0] == 1.0 and np.array_equal(o[0, 0], v[0, 0])


def test_merge_identity_and_undefined():
    rng = np.random.default_rng(1)
    o1 = rng.standard_normal((3, 2, 4)); m1 = rng.standard_normal((3, 2)); s1 = 1 + rng.random((3, 2))
    empty = (np.full((3, 2), -np.inf), np.zeros((3, 2)), np.zeros((3, 2, 4)))
    out, lse = A.merge_partials((m1, s1, o1), empty)
    assert np.allclose(out, o1 / s1[..., None], rtol=0, atol=1e-15)
    assert np.allclose(lse, m1 + np.log(s1))
    with pytest.raises(ValueError):
        A.merge_partials(empty, empty)


def test_merge_commutative_bitwise():
    q, ks, vs, ku, vu = make_attn_inputs(1, 5, 4, 2, 16, 9, 3, seed=7)
    p1 = A.attend_shared(q[0], ks[0], vs[0], 0.25)
    p2 = A.attend_unshared(q[0], ku[0], vu[0], 2, 0.25)
    a, la = A.merge_partials(p1, p2)
    b, lb = A.merge_partials(p2, p1)
    assert np.array_equal(a, b) and np.array_equal(la, lb)


@pytest.mark.parametrize("trial", range(40))
def test_staged_equals_library_attention(trial):     # S:L173 (random shapes)
    rng = np.random.default_rng(100 + trial)
    hkv = int(rng.choice([1, 2, 4])); G = int(rng.choice([1, 2, 4]))
    bw, d, ls, nd = int(rng.integers(1, 7)), int(rng.choice([8, 16, 32])), int(rng.integers(1, 40)), 3
    n = int(rng.integers(0, nd + 1))
    q, ks, vs, ku, vu = make_attn_inputs(1, bw, hkv * G, hkv, d, ls, nd, seed=trial, sigma_q=float(rng.choice([1, 3])))
    scale = 1.0 / math.sqrt(d)
    ref = sdpa_reference(q[0], ks[0], vs[0], ku[0], vu[0], n, scale)
    out, lse = A.staged_attention(q[0], ks[0], vs[0], ku[0], vu[0], n, scale)
    full, flse = A.full_attention(q[0], ks[0], vs[0], ku[0], vu[0], n, scale)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(full, ref, rtol=1e-12, atol=1e-12)
    assert np.allclose(lse, flse, rtol=1e-12, atol=1e-12)


def test_equal_keys_give_mean_of_values():           # closed form: uniform weights
    bw, hq, hkv, d, ls = 2, 2, 1, 8, 5
    rng = np.random.default_rng(3)
    q = rng.standard_normal((bw, hq, d))
    ks = np.repeat(rng.standard_normal((1, hkv, d)), ls, axis=0)
    vs = rng.standard_normal((ls, hkv, d))
    ku = np.repeat(ks[:1][None], bw, axis=0)          # one own token, same key
    vu = rng.standard_normal((bw, 1, hkv, d))
    out, lse = A.staged_attention(q, ks, vs, ku, vu, 1, 0.3)
    for b in range(bw):
        for h in range(hq):
            want = (vs[:, 0, :].sum(0) + vu[b, 0, 0]) / (ls + 1)
            assert np.allclose(out[b, h], want, atol=1e-13)
            assert np.isclose(lse[b, h], 0.3 * q[b, h] @ ks[0, 0] + math.log(ls + 1))


def test_beam_isolation_and_gqa_mapping():           # S:L165; GQA h -> h // G
    q, ks, vs, ku, vu = make_attn_inputs(1, 4, 4, 2, 16, 11, 3, seed=5)
    q, ks, vs, ku, vu = q[0], ks[0], vs[0], ku[0], vu[0]
    base, _ = A.staged_attention(q, ks, vs, ku, vu, 3, 0.25)
    ku2 = ku.copy(); ku2[1] += 1.0
    pert, _ = A.staged_attention(q, ks, vs, ku2, vu, 3, 0.25)
    assert np.array_equal(base[0], pert[0]) and not np.allclose(base[1], pert[1])
    vs2 = vs.copy(); vs2[:, 1, :] += 1.0                # kv head 1 feeds query heads 2, 3 only
    pert, _ = A.staged_attention(q, ks, vs2, ku, vu, 3, 0.25)
    assert np.array_equal(base[:, :2], pert[:, :2]) and not np.allclose(base[:, 2:], pert[:, 2:])


def test_split_prompt_merge_is_exact():              # OnlineSoftmax associativity
    q, ks, vs, ku, vu = make_attn_inputs(1, 3, 2, 1, 16, 30, 3, seed=9)
    q, ks, vs = q[0], ks[0], vs[0]
    whole = A.attend_shared(q, ks, vs, 0.25)
    a = A.attend_shared(q, ks[:13], vs[:13], 0.25)
    b = A.attend_shared(q, ks[13:], vs[13:], 0.25)
    out_ab, lse_ab = A.merge_partials(a, b)
    assert np.allclose(out_ab, whole[2] / whole[1][..., None], atol=1e-13)
    assert np.allclose(lse_ab, whole[0] + np.log(whole[1]), atol=1e-13)
