"""ctypes loader of oracle/paper_heap.c (the paper's heap selection in fp32 C, threaded over
requests): bench.py's cpu_baseline.paper_heap and a selection oracle pinned in
tests/test_paper_heap_c.py.

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py). Built by __graft_entry__.build()
into oracle/lib/libpaper_heap.so; importing raises OSError if it is not built.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libpaper_heap.so")
SRC = os.path.join(HERE, "paper_heap.c")


def build(force: bool = False) -> str:
    import subprocess
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        subprocess.run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", SRC, "-o", LIB, "-lm"],
                       check=True, capture_output=True, text=True)
    return LIB


_lib = ctypes.CDLL(LIB)
_lib.ph_build.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
_lib.ph_build.restype = ctypes.c_void_p
_lib.ph_free.argtypes = [ctypes.c_void_p]
_lib.ph_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.ph_run.restype = ctypes.c_int


class PaperHeap:
    """The item trie built from the oracle's sorted de-duplicated keys (Vocabulary.keys)."""

    def __init__(self, keys: np.ndarray, vocab: int, nd: int):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        self.vocab, self.nd = vocab, nd
        self.h = _lib.ph_build(keys.ctypes.data, keys.shape[0], vocab, nd)
        if not self.h:
            raise MemoryError("ph_build failed")

    def __del__(self):
        if getattr(self, "h", None):
            _lib.ph_free(self.h)
            self.h = None

    def run(self, logits, bw: int, threads: int = 1, top_k: int = 0):
        """logits[r][s]: fp32 [rows_s][V] of request r at step s (rows_0 >= 1, else >= bw).
        Returns dict(parent, token [n][nd][bw] int32, score fp32, n_live [n][nd], visits, cands)."""
        n = len(logits)
        arrs = [np.ascontiguousarray(logits[r][s], dtype=np.float32) for r in range(n) for s in range(self.nd)]
        for a in arrs:
            assert a.ndim == 2 and a.shape[1] == self.vocab
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        par = np.empty((n, self.nd, bw), np.int32)
        tok = np.empty((n, self.nd, bw), np.int32)
        sco = np.empty((n, self.nd, bw), np.float32)
        nl = np.empty((n, self.nd), np.int32)
        st = np.zeros(2, np.int64)
        _lib.ph_run(self.h, n, ptrs, bw, top_k, threads, par.ctypes.data, tok.ctypes.data, sco.ctypes.data,
                    nl.ctypes.data, st.ctypes.data)
        return {"parent": par, "token": tok, "score": sco, "n_live": nl, "visits": int(st[0]),
                "cands": int(st[1]), "visit_frac": float(st[0]) / max(1, int(st[1]))}
