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
    c_all, b_all, v_all = c, b, v
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
    o_pairs = list(zip(b[sel].tolist(), v[sel].tolist()))
    g_pairs = list(zip(np.asarray(g_par[:n_o]).tolist(), np.asarray(g_tok[:n_o]).tolist()))
    c64 = {(int(bb), int(vv)): float(cc) for bb, vv, cc in zip(b_all, v_all, c_all)}
    gs = np.asarray(g_score[:n_o], dtype=np.float64)
    # dead slots
    if np.any(np.asarray(g_par[n_o:]) != -1) or np.any(np.asarray(g_tok[n_o:]) != -1):
        raise ParityFailure(f"{where}: dead slots not (-1, -1)")
    if np.any(~np.isneginf(np.asarray(g_score[n_o:], dtype=np.float64))):
        raise ParityFailure(f"{where}: dead slot scores not -inf")
    for j, p in enumerate(g_pairs):
        if p not in c64:
            raise ParityFailure(f"{where}: slot {j} pair {p} is not a legal candidate")
        if abs(gs[j] - c64[p]) > tol(c64[p]):
            raise ParityFailure(f"{where}: slot {j} score {gs[j]!r} vs fp64 {c64[p]!r}")
    if g_pairs == o_pairs:
        return "strict"
    theta64 = c64[o_pairs[-1]]
    for p in set(g_pairs) ^ set(o_pairs):
        cut = rowcut.get(p[0])
        if abs(c64[p] - theta64) > tol(theta64) and (cut is None or abs(c64[p] - cut) > tol(cut)):
            raise ParityFailure(f"{where}: set differs at {p} (c64 {c64[p]!r}, theta64 {theta64!r})")
    for j in range(n_o - 1):
        a, bnext = c64[g_pairs[j]], c64[g_pairs[j + 1]]
        if bnext > a + tol(a):
            raise ParityFailure(f"{where}: order inversion at slot {j}")
        if bnext == a:
            fa = g_pairs[j][0] * voc.vocab + g_pairs[j][1]
            fb = g_pairs[j + 1][0] * voc.vocab + g_pairs[j + 1][1]
            if not fa < fb:
                raise ParityFailure(f"{where}: tie order at slot {j}")
    return "adjudicated"


def gpu_states(hist_par, hist_tok, scores, nlive):
    """Oracle BeamStates rebuilt from GPU histories: hist_* [t][B][BW] numpy, scores [B][BW]."""
    B = scores.shape[0]
    out = []
    for r in range(B):
        out.append(O.state_from_history([h[r] for h in hist_par], [h[r] for h in hist_tok],
                                        scores[r], int(nlive[r])))
    return out
