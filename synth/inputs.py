"""Seeded synthetic workloads shaped like the paper's.

* Items: N distinct ND-tuples drawn uniformly from [0, V)^ND without replacement. Item i is the
  base-V digit expansion of pi(i), where pi is a keyed Feistel permutation of [0, V^ND) (4 rounds,
  splitmix64 round function, cycle-walking when the domain has an odd number of bits). The paper
  gives no item distribution (section 9.1 uses real datasets), so uniform is a declared
  choice. The list is returned UNSORTED in generation order; `dup_frac` appends duplicates and
  shuffles, to exercise de-duplication.
* Logits: i.i.d. fp32 x = sigma * z, z ~ N(0, 1) from numpy's PCG64 (sigma = 2 "flat", 4 "peaky").
  Multiplying by a power of two is exact, so the bytes are fully determined by (seed, shape, sigma).
* Prefix-keyed logits (tiny exhaustive tests): x(prefix, v) is an Irwin-Hall(4) sum of 16-bit
  fields of splitmix64(seed, request, prefix, v), times 2^-15: exactly representable in fp32 and
  bit-identical in any language.

Nothing here computes any part of the beam-search method.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# BASELINE.json "configs", in order. n_items for C4 is SURVEY.md's proposal (BASELINE gives none).
CONFIGS = {
    "C1": dict(batch=1, beam_width=4, vocab=16, nd=3, n_items=200),
    "C2": dict(batch=64, beam_width=128, vocab=8192, nd=3, n_items=10_000_000),
    "C3": dict(batch=256, beam_width=256, vocab=8192, nd=3, n_items=100_000_000),
    "C4": dict(batch=512, beam_width=512, vocab=16384, nd=4, n_items=100_000_000),
    "C5": dict(batch=128, beam_width=512, vocab=65536, nd=3, n_items=1_000_000_000),
    # C3 with clustered (Zipf s = 1) semantic IDs instead of uniform ones (make_items_clustered)
    "C3Z": dict(batch=256, beam_width=256, vocab=8192, nd=3, n_items=100_000_000, clustered=1.0),
}


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["name"] = name
    c["trie_key"] = config_key(name)
    return c


def splitmix64(x):
    """splitmix64 finaliser on uint64 (numpy array or python int). Wrapping arithmetic."""
    scalar = not isinstance(x, np.ndarray)
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return int(z) if scalar else z


def make_config_items(cfg: dict) -> np.ndarray:
    """The item list of a config: uniform (make_items) or clustered (make_items_clustered)."""
    if cfg.get("clustered"):
        return make_items_clustered(cfg["n_items"], cfg["vocab"], cfg["nd"], cfg["trie_key"], s=cfg["clustered"])
    return make_items(cfg["n_items"], cfg["vocab"], cfg["nd"], cfg["trie_key"])


def config_key(name: str) -> int:
    k = int(name[1:].rstrip("Z")) + (100 if name.endswith("Z") else 0)
    return splitmix64(2512115290 + k)


def _feistel_round_keys(key: int, rounds: int):
    return [np.uint64(splitmix64((key + 0x632BE59BD9B4E019 * (r + 1)) & 0xFFFFFFFFFFFFFFFF))
            for r in range(rounds)]


def feistel_permute(i: np.ndarray, bits: int, key: int, rounds: int = 4) -> np.ndarray:
    """Keyed pseudorandom permutation of [0, 2^bits) applied to uint64 array i (values < 2^bits).

    Feistel network with halves of a = floor(bits/2) and b = bits - a bits (unbalanced when bits
    is odd: the halves swap widths every round). Each round (L, R) -> (R, L ^ F(R)) is invertible,
    so the composition is a bijection of [0, 2^bits) with no cycle walking.
    """
    assert 2 <= bits <= 64 and rounds % 2 == 0
    a = bits // 2
    b = bits - a
    rk = _feistel_round_keys(key, rounds)
    v = np.asarray(i, dtype=np.uint64)
    la, lb = a, b                      # widths of (L, R)
    left = v >> np.uint64(lb)
    right = v & np.uint64((1 << lb) - 1)
    for r in range(rounds):
        f = splitmix64(right ^ rk[r])
        f &= np.uint64((1 << la) - 1)
        left ^= f
        left, right = right, left      # new L has lb bits, new R has la bits
        la, lb = lb, la
    return (left << np.uint64(lb)) | right


def make_items(n: int, vocab: int, nd: int, key: int, dup_frac: float = 0.0,
               shuffle_seed: int | None = None, chunk: int = 1 << 24) -> np.ndarray:
    """N distinct uniform ND-tuples over [0, vocab) as int32 [n (+dups)][nd], unsorted."""
    assert vocab >= 2 and (vocab & (vocab - 1)) == 0, "generator needs a power-of-two vocab"
    b = vocab.bit_length() - 1
    bits = b * nd
    assert n <= (1 << bits), "more items than distinct tuples"
    out = np.empty((n, nd), dtype=np.int32)
    vm = np.uint64(vocab - 1)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        y = feistel_permute(np.arange(s, e, dtype=np.uint64), bits, key)
        for d in range(nd):
            out[s:e, d] = ((y >> np.uint64(b * (nd - 1 - d))) & vm).astype(np.int32)
    if dup_frac > 0.0:
        rng = np.random.default_rng(shuffle_seed if shuffle_seed is not None else key & 0xFFFFFFFF)
        nd_ = max(1, int(n * dup_frac))
        dups = out[rng.integers(0, n, size=nd_)]
        out = np.concatenate([out, dups], axis=0)
        out = out[rng.permutation(out.shape[0])]
        out = np.ascontiguousarray(out)
    return out


def make_items_clustered(n: int, vocab: int, nd: int, key: int, s: float = 1.0, chunk: int = 1 << 24) -> np.ndarray:
    """N distinct ND-tuples with clustered (skewed) prefixes, as int32 [n][nd], unsorted.

    Real semantic IDs are clustered: a few first-level codes hold many items, and under each
    prefix a few next codes dominate (the paper's datasets are out of scope, so
    this is a declared synthetic stand-in). Token d of a tuple is drawn from a Zipf(s) law over
    [0, vocab) whose rank order is permuted per prefix: rank k -> (k * a_p + b_p) mod vocab with
    a_p odd and (a_p, b_p) hashed from the prefix (a bijection, vocab a power of two). Tuples are
    drawn in seeded chunks and de-duplicated keeping first occurrences, until n are distinct.
    """
    assert vocab >= 2 and (vocab & (vocab - 1)) == 0, "generator needs a power-of-two vocab"
    b = vocab.bit_length() - 1
    assert b * nd <= 63
    w = 1.0 / np.arange(1, vocab + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rng = np.random.default_rng(key & 0xFFFFFFFFFFFFFFFF)
    vm = np.uint64(vocab - 1)
    raw = np.zeros(0, dtype=np.uint64)
    while True:
        m = max(4096, (n * 5) // 4 if raw.shape[0] == 0 else (n - uniq.shape[0]) * 2 + 4096)
        parts = []
        for s0 in range(0, m, chunk):
            mm = min(chunk, m - s0)
            h = np.full(mm, np.uint64(key & 0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
            k = np.zeros(mm, dtype=np.uint64)
            for d in range(nd):
                hp = splitmix64(h)
                a = (hp | np.uint64(1)) & vm
                bb = (hp >> np.uint64(32)) & vm
                r = np.minimum(np.searchsorted(cdf, rng.random(mm)).astype(np.uint64), vm)
                with np.errstate(over="ignore"):
                    t = (r * a + bb) & vm
                    h = splitmix64(h ^ (t + np.uint64(0x51ED27 + d)))
                k = (k << np.uint64(b)) | t
            parts.append(k)
        raw = np.concatenate([raw] + parts)
        # first occurrences in draw order
        _, first = np.unique(raw, return_index=True)
        uniq = raw[np.sort(first)]
        if uniq.shape[0] >= n:
            break
    keys_parts = [uniq]
    allk = np.concatenate(keys_parts)[:n]
    out = np.empty((n, nd), dtype=np.int32)
    for d in range(nd):
        out[:, d] = ((allk >> np.uint64(b * (nd - 1 - d))) & vm).astype(np.int32)
    return out


def make_logits(shape, seed: int, sigma: float = 2.0) -> np.ndarray:
    """fp32 i.i.d. N(0, sigma^2) logits of the given shape (numpy PCG64, seeded)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(size=shape, dtype=np.float32)
    x *= np.float32(sigma)
    return x


def make_logits_torch(shape, seed: int, sigma: float = 2.0, device="cuda"):
    """Device-side generator for large bench inputs (torch Philox, seeded). Not bit-equal to
    make_logits; parity at full size D2H-copies what this produced."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    x.mul_(float(sigma))
    return x


def make_logits_rows_torch(requests, rows: int, vocab: int, step: int, key: int, sigma: float = 2.0,
                           col0: int = 0, ncols: int | None = None, device="cuda"):
    """fp32 N(0, sigma^2) logits [len(requests)][rows][ncols] whose values depend only on (key, step,
    request, column): request r's full [rows][vocab] block comes from its own torch Philox stream,
    and columns [col0, col0 + ncols) are kept. A request therefore sees the same bytes however the
    batch is split across ranks (request split) or the columns across shards (codebook shard)."""
    import torch
    ncols = vocab - col0 if ncols is None else ncols
    out = torch.empty((len(requests), rows, ncols), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    for i, r in enumerate(requests):
        seed = splitmix64((key + 0x9E3779B97F4A7C15 * (step + 1) + 0x632BE59BD9B4E019 * (int(r) + 1))
                          & 0xFFFFFFFFFFFFFFFF)
        g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
        x = torch.randn((rows, vocab), generator=g, device=device, dtype=torch.float32)
        out[i].copy_(x[:, col0:col0 + ncols])
        out[i].mul_(float(sigma))
    return out


def prefix_keyed_row(seed: int, request: int, prefix, vocab: int) -> np.ndarray:
    """fp32 row x(prefix, v) for v < vocab: Irwin-Hall(4) of 16-bit fields of a splitmix64 hash,
    scaled by 2^-15 (exact). Same prefix -> same row, whatever slot it sits in."""
    h = splitmix64((seed * 0x9E3779B1 + request) & 0xFFFFFFFFFFFFFFFF)
    for t in prefix:
        h = splitmix64((h ^ (int(t) + 0x51ED27)) & 0xFFFFFFFFFFFFFFFF)
    h = splitmix64((h + len(prefix)) & 0xFFFFFFFFFFFFFFFF)
    v = np.arange(vocab, dtype=np.uint64)
    with np.errstate(over="ignore"):
        r = splitmix64(v ^ np.uint64(h))
    s = np.zeros(vocab, dtype=np.int64)
    for k in range(4):
        s += ((r >> np.uint64(16 * k)) & np.uint64(0xFFFF)).astype(np.int64)
    return ((s - 131070).astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float32)


# ---- staged attention (second workload) ----------------------------------
# Attention-layer shapes of the paper's largest evaluated model family (Qwen3 up to
# 4B; Qwen3-4B: 32 query heads, 8 KV heads, head_dim 128) at the paper's memory-study point
# (input length 1k, BW 256; ND = 3 decode phases).
ATTN_CONFIGS = {
    "A1": dict(n_req=2, bw=4, hq=4, hkv=2, d=128, ls=70, nd=3),          # tiny parity case
    "A2": dict(n_req=16, bw=256, hq=32, hkv=8, d=128, ls=1024, nd=3),    # bench workload
    "A3": dict(n_req=4, bw=512, hq=32, hkv=8, d=128, ls=3072, nd=3),     # BW 512, 3k prompt (L559-566)
}


def to_bf16_grid(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even) and return them as fp32, so both sides
    see the identical bf16 numbers (the CUDA side receives x.view(uint32) >> 16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return r.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns of values already on the bf16 grid (to_bf16_grid)."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def make_attn_inputs(n_req: int, bw: int, hq: int, hkv: int, d: int, ls: int, nd: int, seed: int,
                     sigma_q: float = 1.0):
    """Seeded bf16-grid inputs of one decode step's attention layer (values as fp32 arrays):
    q [n_req][bw][hq][d] ~ sigma_q N(0,1); shared k, v [n_req][ls][hkv][d] ~ N(0,1) (the prompt's
    KV after prefill, token-major); unshared k, v [n_req][bw][nd][hkv][d] ~ N(0,1) (each beam's
    generated tokens: capacity BW x ND)."""
    rng = np.random.default_rng(seed)
    g = lambda *s: to_bf16_grid(rng.standard_normal(size=s, dtype=np.float32))
    q = to_bf16_grid(rng.standard_normal(size=(n_req, bw, hq, d), dtype=np.float32) * np.float32(sigma_q))
    ks, vs = g(n_req, ls, hkv, d), g(n_req, ls, hkv, d)
    ku, vu = g(n_req, bw, nd, hkv, d), g(n_req, bw, nd, hkv, d)
    return q, ks, vs, ku, vu
