"""Staged shared/unshared decode attention (second workload) --
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

PAPER.md L339 (section 5.2, "Staged Computation Allocation"): "xAttention divides the attention
computation with common prefixes into a shared stage and an unshared stage ... computes the local
attention scores and statistics (i.e., local maxima and sums) for the shared and unshared stages
independently. It then applies OnlineSoftmax to produce the final logits". PAPER.md L324: the
shared cache holds the prompt's KV once (from prefill), the unshared cache holds each beam's
generated tokens (capacity BW x ND). SPEC.md S:L136-179 fixes the operations:

  attend_shared(q, ks, vs, scale)        partial (m, s, o) of every (beam, head) over all prompt
                                         positions
  attend_unshared(q, ku, vu, n, scale)   partial over each beam's own first n generated tokens
                                         
  merge_partials(p1, p2)                 m = max(m1, m2), w_i = exp(m_i - m),
                                         out = (o1 w1 + o2 w2) / (s1 w1 + s2 w2)
  full_attention(q, ks, vs, ku, vu, n, scale)
                                         the plain definition: softmax attention of beam b over
                                         the concatenation prompt + b's own tokens

Partials follow S:L136-139: m = max of the scaled logits, s = sum exp(logit - m),
o = sum exp(logit - m) v (unnormalised); an empty stage is (m = -inf, s = 0, o = 0).
Grouped-query attention: query head h reads KV head h // (hq / hkv) (the Qwen3 layout of the
paper's models). Everything is fp64 numpy, one (beam, head) at a time.

Shapes: q [bw][hq][d]; ks, vs [ls][hkv][d]; ku, vu [bw][nd][hkv][d]. One request at a time.
Parity status: pinned (tests/test_attn_oracle.py).
"""
import numpy as np

NEG_INF = -np.inf


def _kv_head(h: int, hq: int, hkv: int) -> int:
    return h // (hq // hkv)


def _partial(qv: np.ndarray, keys: np.ndarray, vals: np.ndarray, scale: float):
    """(m, s, o) of one query over keys [n][d], vals [n][d], fp64."""
    d = qv.shape[0]
    if keys.shape[0] == 0:
        return NEG_INF, 0.0, np.zeros(d)
    logits = (keys.astype(np.float64) @ qv.astype(np.float64)) * scale
    m = float(np.max(logits))
    w = np.exp(logits - m)
    return m, float(np.sum(w)), w @ vals.astype(np.float64)


def attend_shared(q, ks, vs, scale):
    """every (beam, head) against every prompt position; returns m, s [bw][hq] and
    o [bw][hq][d]."""
    bw, hq, d = q.shape
    hkv = ks.shape[1]
    m = np.empty((bw, hq)); s = np.empty((bw, hq)); o = np.empty((bw, hq, d))
    for b in range(bw):
        for h in range(hq):
            g = _kv_head(h, hq, hkv)
            m[b, h], s[b, h], o[b, h] = _partial(q[b, h], ks[:, g, :], vs[:, g, :], scale)
    return m, s, o


def attend_unshared(q, ku, vu, n, scale):
    """beam b attends only its own generated tokens t < n."""
    bw, hq, d = q.shape
    hkv = ku.shape[2]
    m = np.empty((bw, hq)); s = np.empty((bw, hq)); o = np.empty((bw, hq, d))
    for b in range(bw):
        for h in range(hq):
            g = _kv_head(h, hq, hkv)
            m[b, h], s[b, h], o[b, h] = _partial(q[b, h], ku[b, :n, g, :], vu[b, :n, g, :], scale)
    return m, s, o


def merge_partials(p1, p2):
    """S:L167-174 (OnlineSoftmax merge): returns (out, lse) with
    lse = m + ln(s1 w1 + s2 w2) the log-sum-exp of all scaled logits. Both empty -> ValueError."""
    m1, s1, o1 = p1
    m2, s2, o2 = p2
    m1 = np.asarray(m1, dtype=np.float64); m2 = np.asarray(m2, dtype=np.float64)
    if np.any(np.isneginf(m1) & np.isneginf(m2)):
        raise ValueError("undefined attention: both partials empty")
    m = np.maximum(m1, m2)
    w1 = np.where(np.isneginf(m1), 0.0, np.exp(m1 - m))
    w2 = np.where(np.isneginf(m2), 0.0, np.exp(m2 - m))
    den = s1 * w1 + s2 * w2
    out = (o1 * w1[..., None] + o2 * w2[..., None]) / den[..., None]
    return out, m + np.log(den)


def full_attention(q, ks, vs, ku, vu, n, scale):
    """S:L175-179, the plain definition: out[b][h] = softmax_j(scale * q[b][h] . k_j) v_j over
    j in prompt positions followed by beam b's own tokens t < n. Returns (out, lse)."""
    bw, hq, d = q.shape
    hkv = ks.shape[1]
    out = np.empty((bw, hq, d)); lse = np.empty((bw, hq))
    for b in range(bw):
        for h in range(hq):
            g = _kv_head(h, hq, hkv)
            keys = np.concatenate([ks[:, g, :], ku[b, :n, g, :]]).astype(np.float64)
            vals = np.concatenate([vs[:, g, :], vu[b, :n, g, :]]).astype(np.float64)
            logits = keys @ q[b, h].astype(np.float64) * scale
            mx = np.max(logits)
            p = np.exp(logits - mx)
            out[b, h] = (p / p.sum()) @ vals
            lse[b, h] = mx + np.log(p.sum())
    return out, lse


def staged_attention(q, ks, vs, ku, vu, n, scale):
    """The staged computation of PAPER.md L339: shared stage, unshared stage, merge."""
    return merge_partials(attend_shared(q, ks, vs, scale), attend_unshared(q, ku, vu, n, scale))
