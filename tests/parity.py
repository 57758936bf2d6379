"""Parity protocol between the CUDA path and the oracle.

Teacher forcing (reading R15): the oracle's step t consumes the GPU state after step t-1
(prefixes from the GPU's parent/token histories, the GPU's fp32 scores widened to fp64), so one
adjudicated near-tie does not cascade. Comparison of one request's step:
  1. n_live equal;
  2. (parent, token) equal element-wise -> scores within tol(s) = 1e-5 * max(1, |s|) -> PASS;
  3. otherwise adjudicate (north_star: "candidates whose score lies within 1e-5 of the k-th
     threshold are adjudicated by the oracle's fp64 recompute"): every pair in G \\ O and O \\ G
     has |c64 - theta64| <= tol(theta64); selected fp64 scores are non-increasing within tol;
     GPU scores within tol of their fp64 recompute.
With a per-beam Top-K (NEXT f3) the oracle truncates each row to its K best first; a pair may
then also differ when it lies within tol of its row's K-th fp64 score (the row cut, the same
near-tie adjudication applied at the per-row boundary).
"""
from __future__ import annotations

import numpy as np

from oracle import xbeam_oracle as O


def tol(s: float) -> float:
    return 1e-5 * max(1.0, abs(float(s)))


class ParityFailure(AssertionError):
    pass


def compare_step(voc, state, logits_r, bw, g_par, g_tok, g_score, g_nlive, where="", top_k=None):
    """Returns 'strict' or 'adjudicated'; raises ParityFailure otherwise."""
    c, flat, b, v, nonfinite = O.step_candidates(voc, state, logits_r)
    c_all, flat_all = c, flat          # flat is ascending (rows in slot order, tokens sorted)
    V = voc.vocab
    rowcut = {}
    if top_k is not None and top_k < bw:
        keep = O.per_beam_topk(c, flat, b, top_k)
        for bb in np.unique(b):
            m = b[keep] == bb
            if np.count_nonzero(b == bb) > top_k:
                rowcut[int(bb)] = float(np.min(c[keep][m]))
        c, flat, b, v = c[keep], flat[keep], b[keep], v[keep]
    sel = O.select_top_bw(c, flat, bw)
    n_o = len(sel)
    if int(g_nlive) != n_o:
        raise ParityFailure(f"{where}: n_live gpu {g_nlive} != oracle {n_o}")
    o_flat = flat[sel]
    gp = np.asarray(g_par[:n_o], dtype=np.int64)
    gt = np.asarray(g_tok[:n_o], dtype=np.int64)
    # dead slots
    if np.any(np.asarray(g_par[n_o:]) != -1) or np.any(np.asarray(g_tok[n_o:]) != -1):
        raise ParityFailure(f"{where}: dead slots not (-1, -1)")
    if np.any(~np.isneginf(np.asarray(g_score[n_o:], dtype=np.float64))):
        raise ParityFailure(f"{where}: dead slot scores not -inf")
    # every GPU pair must be a legal candidate (b < n_live, v among the children of b's prefix)
    g_flat = gp * V + gt
    ok = (gp >= 0) & (gp < state.n_live) & (gt >= 0) & (gt < V)
    pos = np.clip(np.searchsorted(flat_all, g_flat), 0, max(len(flat_all) - 1, 0))
    ok &= flat_all[pos] == g_flat
    if not np.all(ok):
        j = int(np.argmin(ok))
        raise ParityFailure(f"{where}: slot {j} pair {(int(gp[j]), int(gt[j]))} is not a legal candidate")
    g_c64 = c_all[pos]                   # fp64 recompute of each GPU selection
    gs = np.asarray(g_score[:n_o], dtype=np.float64)
    tol_v = 1e-5 * np.maximum(1.0, np.abs(g_c64))
    bad = ~(np.abs(gs - g_c64) <= tol_v)
    if np.any(bad):
        j = int(np.argmax(bad))
        raise ParityFailure(f"{where}: slot {j} score {gs[j]!r} vs fp64 {g_c64[j]!r}")
    if np.array_equal(g_flat, o_flat):
        return "strict"
    theta64 = float(c[sel][-1])

    def c64_of(f):
        return float(c_all[np.searchsorted(flat_all, f)])

    for f in set(g_flat.tolist()) ^ set(o_flat.tolist()):
        cc = c64_of(f)
        cut = rowcut.get(f // V)
        if abs(cc - theta64) > tol(theta64) and (cut is None or abs(cc - cut) > tol(cut)):
            raise ParityFailure(f"{where}: set differs at {(f // V, f % V)} (c64 {cc!r}, theta64 {theta64!r})")
    for j in range(n_o - 1):
        a, bnext = g_c64[j], g_c64[j + 1]
        if bnext > a + tol(a):
            raise ParityFailure(f"{where}: order inversion at slot {j}")
        if bnext == a and not g_flat[j] < g_flat[j + 1]:
            raise ParityFailure(f"{where}: tie order at slot {j}")
    return "adjudicated"


def compare_many(voc, states, logits_fn, bw, par, tok, sc, nl, reqs, where="", top_k=None, threads=None):
    """compare_step over many requests on a thread pool (numpy releases the GIL in its kernels).
    states: {r: BeamState}; logits_fn(r) -> that request's [rows][ld] logits (fp32 numpy).
    Returns {'strict': n, 'adjudicated': n, 'adjudicated_at': [(r, ...)]}."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or min(32, max(1, len(os.sched_getaffinity(0))))

    def one(r):
        return r, compare_step(voc, states[r], logits_fn(r), bw, par[r], tok[r], sc[r], nl[r],
                               where=f"{where} req {r}", top_k=top_k)

    out = {"strict": 0, "adjudicated": 0, "adjudicated_at": []}
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for r, res in ex.map(one, reqs):
            out[res] += 1
            if res == "adjudicated":
                out["adjudicated_at"].append(r)
    return out


def gpu_states(hist_par, hist_tok, scores, nlive):
    """Oracle BeamStates rebuilt from GPU histories: hist_* [t][B][BW] numpy, scores [B][BW]."""
    B = scores.shape[0]
    out = []
    for r in range(B):
        out.append(O.state_from_history([h[r] for h in hist_par], [h[r] for h in hist_tok],
                                        scores[r], int(nlive[r])))
    return out
