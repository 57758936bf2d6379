"""Thin ctypes binding over libxgr_beam.so (include/xgr_beam.h). Argument marshalling only:
every step of the path runs in the library's CUDA kernels. torch is used for device memory and
streams. There is no CPU fallback: if the library is missing this module fails to import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# XGR_LIB: an alternative build of the same library (development A/B builds only)
LIB_PATH = os.environ.get("XGR_LIB") or os.path.join(_HERE, "lib", "libxgr_beam.so")

XGR_OK = 0
STATUS_NAMES = {
    0: "XGR_OK", 1: "XGR_ERR_INVALID_ARG", 2: "XGR_ERR_UNSUPPORTED", 3: "XGR_ERR_TOKEN_RANGE",
    4: "XGR_ERR_EMPTY_VOCAB", 5: "XGR_ERR_SEQUENCE", 6: "XGR_ERR_ALIGNMENT",
    7: "XGR_ERR_NONFINITE", 8: "XGR_ERR_CUDA", 9: "XGR_ERR_NCCL", 10: "XGR_ERR_OOM",
}
XGR_CFG_NO_PRUNE = 0x1
XGR_CFG_COUNTERS = 0x2
XGR_CFG_NO_SPARSE_KERNEL = 0x4
XGR_CFG_TIMING = 0x8
XGR_CFG_PAPER_HEAP = 0x10   # baseline: the paper's per-beam Top-K lists + sequential heap
XGR_NUM_COUNTERS = 8
COUNTER_NAMES = ["rows_read", "rows_skip_pre", "rows_skip_post", "legal", "survivors",
                 "overflow", "sparse_cands", "dense_steps"]

# every symbol include/xgr_beam.h declares
EXPORTS = ["xgr_beam_init", "xgr_mask_build", "xgr_beam_step", "xgr_beam_step_ex", "xgr_beam_finalize",
           "xgr_beam_destroy", "xgr_last_error", "xgr_abi_version", "xgr_beam_view",
           "xgr_beam_history", "xgr_beam_request_status", "xgr_mask_children", "xgr_mask_info",
           "xgr_beam_counters", "xgr_beam_account", "xgr_beam_launch_count",
           "xgr_beam_kernel_times", "xgr_beam_outputs", "xgr_shard_stats", "xgr_shard_select",
           "xgr_shard_merge", "xgr_kv_reorder", "xgr_beam_step_head", "xgr_beam_next_route",
           "xgr_attn_staged", "xgr_attn_shared", "xgr_attn_unshared", "xgr_attn_merge",
           "xgr_beam_step_host"]

ABI_VERSION = 2

# xgr_config.dev_alloc / dev_free
DEV_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
DEV_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class XgrConfig(ctypes.Structure):
    _fields_ = [
        ("vocab", ctypes.c_int32), ("nd", ctypes.c_int32), ("beam_width", ctypes.c_int32),
        ("top_k", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("device", ctypes.c_int32),
        ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
        ("survivor_cap", ctypes.c_int32), ("theta_rows", ctypes.c_int32),
        ("flags", ctypes.c_uint32), ("dev_alloc", DEV_ALLOC_FN), ("dev_free", DEV_FREE_FN),
        ("alloc_user", ctypes.c_void_p), ("reserved", ctypes.c_int32 * 5),
    ]


class XgrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (the CUDA library is required; there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "xgr_beam_init": [P(XgrConfig), P(VP)],
        "xgr_mask_build": [VP, VP, I64, VP],
        "xgr_beam_step": [VP, I32, VP, I32, I64, VP],
        "xgr_beam_step_ex": [VP, I32, VP, I32, I32, I64, VP],
        "xgr_beam_step_host": [VP, I32, VP, I32, I32, I64, VP],
        "xgr_beam_finalize": [VP, VP, VP, VP, VP, I32, VP],
        "xgr_beam_destroy": [VP],
        "xgr_beam_view": [VP, P(VP), P(VP), P(VP), P(VP), P(VP)],
        "xgr_beam_history": [VP, I32, P(VP), P(VP)],
        "xgr_beam_request_status": [VP, VP, I32, VP],
        "xgr_mask_children": [VP, VP, I32, I64, VP, VP, I64, VP],
        "xgr_mask_info": [VP, VP, VP, VP, VP, VP],
        "xgr_beam_counters": [VP, VP, VP],
        "xgr_beam_account": [VP, VP, VP, VP, VP],
        "xgr_beam_kernel_times": [VP, VP, VP, I32, VP],
        "xgr_beam_outputs": [VP, P(VP), P(VP), P(VP), P(VP)],
        "xgr_shard_stats": [VP, I32, VP, I32, I64, VP, P(VP)],
        "xgr_shard_select": [VP, VP, VP, P(VP), P(VP)],
        "xgr_shard_merge": [VP, VP, VP, VP],
        "xgr_kv_reorder": [VP, I32, I32, I32, I64, I64, I64, I64, VP, I32, VP],
        "xgr_beam_step_head": [VP, I32, VP, I32, I64, VP, I64, VP, I32, VP],
        "xgr_beam_next_route": [VP, VP],
        "xgr_attn_staged": [VP, VP, VP, I32, VP, VP, I64, I64, I32, VP, VP, I32, I32, I32, I32, I32,
                            ctypes.c_float, VP],
        "xgr_attn_shared": [VP, VP, VP, I32, VP, VP, VP, I32, I32, I32, I32, I32, ctypes.c_float, VP],
        "xgr_attn_unshared": [VP, VP, VP, I64, I64, I32, VP, VP, VP, I32, I32, I32, I32, I32,
                              ctypes.c_float, VP],
        "xgr_attn_merge": [VP, VP, VP, VP, VP, VP, I64, I32, VP, VP, VP],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.xgr_last_error.argtypes = []
    lib.xgr_last_error.restype = ctypes.c_char_p
    lib.xgr_beam_launch_count.argtypes = [VP]
    lib.xgr_beam_launch_count.restype = ctypes.c_int64
    lib.xgr_abi_version.argtypes = []
    lib.xgr_abi_version.restype = ctypes.c_int32
    if lib.xgr_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.xgr_abi_version()}, binding expects {ABI_VERSION} "
                          "(rebuild: python -c 'import __graft_entry__ as g; g.build()')")
    return lib


lib = _load()


def _check(st: int):
    if st != XGR_OK:
        raise XgrError(st, lib.xgr_last_error().decode(errors="replace"))


def last_error() -> str:
    return lib.xgr_last_error().decode(errors="replace")


# ---- thin wrappers with the C names -------------------------------------------------------------
def xgr_beam_init(cfg: XgrConfig) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.xgr_beam_init(ctypes.byref(cfg), ctypes.byref(h)))
    return h


def xgr_mask_build(ctx, items: np.ndarray, stream=0):
    items = np.ascontiguousarray(items, dtype=np.int32)
    n = items.shape[0] if items.ndim >= 1 else 0
    _check(lib.xgr_mask_build(ctx, items.ctypes.data if n else None, n, stream))


def xgr_beam_step(ctx, batch, logits_ptr, rows, ld, stream=0):
    _check(lib.xgr_beam_step(ctx, batch, logits_ptr, rows, ld, stream))


XGR_DTYPE_F32, XGR_DTYPE_BF16 = 0, 1


def xgr_beam_step_ex(ctx, batch, logits_ptr, dtype, rows, ld, stream=0):
    _check(lib.xgr_beam_step_ex(ctx, batch, logits_ptr, dtype, rows, ld, stream))


def xgr_beam_step_host(ctx, batch, host_ptr, dtype, rows, ld, stream=0):
    _check(lib.xgr_beam_step_host(ctx, batch, host_ptr, dtype, rows, ld, stream))


def xgr_beam_finalize(ctx, tokens, item_rank, score, n_live, outputs_on_device, stream=0):
    return lib.xgr_beam_finalize(ctx, tokens, item_rank, score, n_live, outputs_on_device, stream)


def xgr_beam_destroy(ctx):
    _check(lib.xgr_beam_destroy(ctx))


def xgr_mask_children(ctx, prefixes: np.ndarray, depth: int, cap: int, stream=0):
    prefixes = np.ascontiguousarray(prefixes, dtype=np.int32).reshape(-1, max(depth, 1))
    n = prefixes.shape[0] if depth > 0 else prefixes.shape[0]
    counts = np.zeros(n, dtype=np.int32)
    toks = np.zeros((n, max(cap, 1)), dtype=np.int32)
    _check(lib.xgr_mask_children(ctx, prefixes.ctypes.data if depth > 0 else None, depth, n,
                                 counts.ctypes.data, toks.ctypes.data, cap, stream))
    return counts, toks[:, :cap]


def xgr_mask_info(ctx, nd: int):
    n = ctypes.c_int64()
    nodes = np.zeros(nd + 1, np.int64)
    dense = np.zeros(nd + 1, np.int64)
    maxc = np.zeros(nd + 1, np.int64)
    b = ctypes.c_int64()
    _check(lib.xgr_mask_info(ctx, ctypes.byref(n), nodes.ctypes.data, dense.ctypes.data,
                             maxc.ctypes.data, ctypes.byref(b)))
    return {"n_items": n.value, "nodes": nodes, "dense": dense, "max_children": maxc,
            "bytes": b.value}


# ---- zero-copy torch views of library-owned device buffers --------------------------------------
class _CudaArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _view(ptr, shape, typestr, device):
    import torch
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


class BeamSearch:
    """xBeam decode-step selection for one in-flight batch (wraps one xgr_ctx).

    Usage: bs = BeamSearch(V, ND, BW, max_batch); bs.mask_build(items);
           for t in range(ND): bs.step(logits_t); out = bs.finalize()
    """

    def __init__(self, vocab: int, nd: int, beam_width: int, max_batch: int, device: int = 0,
                 flags: int = 0, survivor_cap: int = 0, theta_rows: int = 0, top_k: int = 0,
                 nranks: int = 1, rank: int = 0, allocator=None):
        """allocator: None (cudaMalloc) or "torch": the ctx's device memory comes from torch's
        caching allocator (xgr_config.dev_alloc / dev_free)."""
        import torch
        self.vocab, self.nd, self.bw, self.max_batch = vocab, nd, beam_width, max_batch
        self.device = torch.device("cuda", device)
        cfg = XgrConfig()
        self.alloc_calls = [0, 0]   # (allocations, frees) through the hooks
        if allocator == "torch":
            def _alloc(nbytes, _user):
                self.alloc_calls[0] += 1
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), device)
                except RuntimeError:
                    return None   # -> XGR_ERR_OOM

            def _free(ptr, _user):
                self.alloc_calls[1] += 1
                torch.cuda.caching_allocator_delete(ptr)

            # the callbacks must outlive the ctx
            self._hooks = (DEV_ALLOC_FN(_alloc), DEV_FREE_FN(_free))
            cfg.dev_alloc, cfg.dev_free = self._hooks
        elif allocator is not None:
            raise ValueError("allocator must be None or 'torch'")
        cfg.vocab, cfg.nd, cfg.beam_width, cfg.top_k = vocab, nd, beam_width, top_k
        cfg.max_batch, cfg.device, cfg.nranks, cfg.rank = max_batch, device, nranks, rank
        self.nranks, self.rank = nranks, rank
        cfg.survivor_cap, cfg.theta_rows, cfg.flags = survivor_cap, theta_rows, flags
        self.ctx = xgr_beam_init(cfg)
        self.batch = None
        self.t = 0

    def close(self):
        if self.ctx:
            xgr_beam_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream(stream=None):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def mask_build(self, items: np.ndarray, stream=None):
        xgr_mask_build(self.ctx, items, self._stream(stream))

    def info(self):
        return xgr_mask_info(self.ctx, self.nd)

    def children(self, prefixes, depth: int, cap: int):
        return xgr_mask_children(self.ctx, np.asarray(prefixes), depth, cap, self._stream())

    def step(self, logits, stream=None):
        """logits: fp32 or bf16 [batch][rows][ld] (or [batch][rows][V]); CUDA tensor
        (xgr_beam_step_ex), or a CPU tensor -- pinned for an asynchronous copy -- which the library
        copies into its device staging buffer on the same stream (xgr_beam_step_host)."""
        import torch
        if logits.dim() != 3 or logits.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("logits must be fp32 or bf16 [batch][rows][ld]")
        if logits.stride(2) != 1 or logits.stride(0) != logits.stride(1) * logits.shape[1]:
            raise ValueError("logits must be row-major [batch][rows][ld] (unit column stride)")
        b, rows = logits.shape[0], logits.shape[1]
        dt = XGR_DTYPE_BF16 if logits.dtype == torch.bfloat16 else XGR_DTYPE_F32
        step = xgr_beam_step_ex if logits.is_cuda else xgr_beam_step_host
        step(self.ctx, b, ctypes.c_void_p(logits.data_ptr()), dt, rows, logits.stride(1), self._stream(stream))
        self.batch = b
        self.t += 1

    def next_is_sparse(self) -> bool:
        """Whether the next step takes the sparse route (xgr_beam_next_route)."""
        v = ctypes.c_int32()
        _check(lib.xgr_beam_next_route(self.ctx, ctypes.byref(v)))
        return bool(v.value)

    def step_head(self, hidden, head, bias=None, stream=None):
        """LM-head fusion at a sparse step (NEXT f4; xgr_beam_step_head): hidden CUDA bf16
        [batch][rows][ldh], head CUDA bf16 [V][ldw] (only the first d = hidden.shape[2] columns
        are used if the last dims are views), bias CUDA fp32 [V] or None."""
        import torch
        if hidden.dim() != 3 or hidden.dtype != torch.bfloat16 or hidden.stride(2) != 1:
            raise ValueError("hidden must be bf16 [batch][rows][d] with unit column stride")
        if head.dim() != 2 or head.dtype != torch.bfloat16 or head.stride(1) != 1:
            raise ValueError("head must be bf16 [V][d] with unit column stride")
        if bias is not None and (bias.dtype != torch.float32 or not bias.is_contiguous()):
            raise ValueError("bias must be contiguous fp32 [V]")
        b, rows, d = hidden.shape
        if hidden.stride(0) != hidden.stride(1) * rows:
            raise ValueError("hidden must be row-major [batch][rows][ldh]")
        _check(lib.xgr_beam_step_head(self.ctx, b, ctypes.c_void_p(hidden.data_ptr()), rows, hidden.stride(1),
                                      ctypes.c_void_p(head.data_ptr()), head.stride(0),
                                      ctypes.c_void_p(bias.data_ptr() if bias is not None else 0), d,
                                      self._stream(stream)))
        self.batch = b
        self.t += 1

    # ---- codebook shard phases (nranks > 1): the caller all-gathers between them ----------------
    def shard_stats(self, logits, stream=None):
        """logits: this rank's columns, CUDA fp32 [batch][rows][ld]. Returns a [batch][BW][2]
        fp32 view of the local (m, Z) per row (valid until the next shard call)."""
        import torch
        b, rows = logits.shape[0], logits.shape[1]
        p = ctypes.c_void_p()
        _check(lib.xgr_shard_stats(self.ctx, b, ctypes.c_void_p(logits.data_ptr()), rows,
                                   logits.stride(1), self._stream(stream), ctypes.byref(p)))
        self.batch = b
        self._shard_logits = logits   # must stay alive until shard_select completes
        return _view(p.value, (b, self.bw, 2), "<f4", self.device)

    def shard_select(self, gstats, stream=None):
        """gstats: CUDA fp32 [nranks][batch][BW][2] (all ranks' stats, rank-major). Returns
        (recs uint64-as-int64 [batch][BW], rec_n int32 [batch]) views."""
        r, n = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.xgr_shard_select(self.ctx, ctypes.c_void_p(gstats.data_ptr()), self._stream(stream),
                                    ctypes.byref(r), ctypes.byref(n)))
        return (_view(r.value, (self.batch, self.bw), "<i8", self.device),
                _view(n.value, (self.batch,), "<i4", self.device))

    def shard_merge(self, grecs, grec_n=None, stream=None):
        """grecs int64 [nranks][batch][BW] (all ranks, rank-major); grec_n int32 [nranks][batch] or
        None (the merge counts each rank's nonzero keys: no third collective)."""
        _check(lib.xgr_shard_merge(self.ctx, ctypes.c_void_p(grecs.data_ptr()),
                                   ctypes.c_void_p(0 if grec_n is None else grec_n.data_ptr()),
                                   self._stream(stream)))
        self.t += 1
        self._shard_logits = None

    def finalize_in_place(self, stream=None):
        """Ends the batch without copying: results stay in the ctx buffers (outputs_view())."""
        _check(xgr_beam_finalize(self.ctx, None, None, None, None, 1, self._stream(stream)))
        self.t = 0

    def finalize(self, on_device: bool = True, stream=None, out=None):
        """Returns dict(tokens [B][BW][ND] int32, item_rank [B][BW] int64, score [B][BW] fp32,
        n_live [B] int32); CUDA tensors if on_device else numpy arrays (pinned copies)."""
        import torch
        B = self.batch
        if B is None:
            _check(xgr_beam_finalize(self.ctx, None, None, None, None, 1, self._stream(stream)))
        if on_device:
            if out is None:
                out = {
                    "tokens": torch.empty((B, self.bw, self.nd), dtype=torch.int32, device=self.device),
                    "item_rank": torch.empty((B, self.bw), dtype=torch.int64, device=self.device),
                    "score": torch.empty((B, self.bw), dtype=torch.float32, device=self.device),
                    "n_live": torch.empty((B,), dtype=torch.int32, device=self.device),
                }
            st = xgr_beam_finalize(self.ctx, ctypes.c_void_p(out["tokens"].data_ptr()),
                                   ctypes.c_void_p(out["item_rank"].data_ptr()),
                                   ctypes.c_void_p(out["score"].data_ptr()),
                                   ctypes.c_void_p(out["n_live"].data_ptr()), 1, self._stream(stream))
        else:
            if out is None:
                out = {
                    "tokens": np.empty((B, self.bw, self.nd), dtype=np.int32),
                    "item_rank": np.empty((B, self.bw), dtype=np.int64),
                    "score": np.empty((B, self.bw), dtype=np.float32),
                    "n_live": np.empty((B,), dtype=np.int32),
                }
            st = xgr_beam_finalize(self.ctx, out["tokens"].ctypes.data, out["item_rank"].ctypes.data,
                                   out["score"].ctypes.data, out["n_live"].ctypes.data, 0,
                                   self._stream(stream))
        self.t = 0
        if st != XGR_OK:
            err = XgrError(st, last_error())
            err.outputs = out
            raise err
        return out

    # ---- views for parity tests (zero-copy, valid until the next step/finalize) ----------------
    def view(self):
        p, tk, sc, nl, nd = (ctypes.c_void_p() for _ in range(5))
        _check(lib.xgr_beam_view(self.ctx, ctypes.byref(p), ctypes.byref(tk), ctypes.byref(sc),
                                 ctypes.byref(nl), ctypes.byref(nd)))
        B, BW = self.batch, self.bw
        return {
            "parent": _view(p.value, (B, BW), "<i4", self.device),
            "token": _view(tk.value, (B, BW), "<i4", self.device),
            "score": _view(sc.value, (B, BW), "<f4", self.device),
            "n_live": _view(nl.value, (B,), "<i4", self.device),
            # uint32 node ids read as int32 (dead slots hold 0xFFFFFFFF -> -1)
            "node": _view(nd.value, (B, BW), "<i4", self.device),
        }

    def history(self, step: int):
        p, tk = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.xgr_beam_history(self.ctx, step, ctypes.byref(p), ctypes.byref(tk)))
        B, BW = self.batch, self.bw
        return _view(p.value, (B, BW), "<i4", self.device), _view(tk.value, (B, BW), "<i4", self.device)

    def request_status(self):
        fl = np.zeros(self.batch, dtype=np.uint32)
        _check(lib.xgr_beam_request_status(self.ctx, fl.ctypes.data, self.batch, self._stream()))
        return fl

    def counters(self):
        out = np.zeros(XGR_NUM_COUNTERS, dtype=np.uint64)
        _check(lib.xgr_beam_counters(self.ctx, out.ctypes.data, self._stream()))
        return dict(zip(COUNTER_NAMES, (int(v) for v in out)))

    def outputs_view(self):
        """Zero-copy CUDA views of the ctx-owned final outputs (written by the last step)."""
        t, r, sc, nl = (ctypes.c_void_p() for _ in range(4))
        _check(lib.xgr_beam_outputs(self.ctx, ctypes.byref(t), ctypes.byref(r), ctypes.byref(sc),
                                    ctypes.byref(nl)))
        B, BW = self.batch, self.bw
        return {"tokens": _view(t.value, (B, BW, self.nd), "<i4", self.device),
                "item_rank": _view(r.value, (B, BW), "<i8", self.device),
                "score": _view(sc.value, (B, BW), "<f4", self.device),
                "n_live": _view(nl.value, (B,), "<i4", self.device)}

    def launch_count(self) -> int:
        return int(lib.xgr_beam_launch_count(self.ctx))

    def kernel_times(self, cap: int = 4096):
        ms = np.zeros(cap, np.float32)
        st = np.zeros(cap, np.int32)
        n = ctypes.c_int32()
        _check(lib.xgr_beam_kernel_times(self.ctx, ms.ctypes.data, st.ctypes.data, cap, ctypes.byref(n)))
        return ms[: n.value], st[: n.value]

    def account(self):
        a, f, lg = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib.xgr_beam_account(self.ctx, ctypes.byref(a), ctypes.byref(f), ctypes.byref(lg),
                                    self._stream()))
        return {"alg_bytes": a.value, "full_bytes": f.value, "legal": lg.value}


def kv_reorder(cache, src, stream=None):
    """In-place KV-cache reorder after a step (xgr_kv_reorder):
    cache[r, p, j, :] <- cache[r, p, src[r, j], :] for src >= 0 and src != j.
    cache: CUDA tensor [n_req][n_panel][bw][E] (last dim contiguous, rows 16-byte multiples);
    src: CUDA int32 [n_req][>= bw], e.g. BeamSearch.view()["parent"]."""
    import torch
    if cache.dim() != 4 or cache.stride(3) != 1:
        raise ValueError("cache must be [n_req][n_panel][bw][E] with a contiguous last dim")
    if src.dtype != torch.int32 or src.dim() != 2 or src.stride(1) != 1:
        raise ValueError("src must be int32 [n_req][>= bw] with unit column stride")
    es = cache.element_size()
    n_req, n_panel, bw, e = cache.shape
    st = torch.cuda.current_stream() if stream is None else stream
    _check(lib.xgr_kv_reorder(ctypes.c_void_p(cache.data_ptr()), n_req, n_panel, bw, e * es,
                              cache.stride(2) * es, cache.stride(1) * es, cache.stride(0) * es,
                              ctypes.c_void_p(src.data_ptr()), src.stride(0), ctypes.c_void_p(st.cuda_stream)))


# ---- staged shared/unshared attention (xgr_attn_*) ----------
def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _attn_shapes(q, ks):
    import torch
    if q.dtype != torch.bfloat16 or q.dim() != 4 or not q.is_contiguous():
        raise ValueError("q must be contiguous bf16 [n_req][bw][hq][d]")
    n_req, bw, hq, d = q.shape
    if ks is not None and (ks.dtype != torch.bfloat16 or ks.dim() != 4 or not ks.is_contiguous()
                           or ks.shape[0] != n_req or ks.shape[3] != d):
        raise ValueError("shared k/v must be contiguous bf16 [n_req][ls][hkv][d]")
    return n_req, bw, hq, d


def _unshared_strides(ku):
    """ku: bf16 view [n_req][bw][>= n][hkv][d] with contiguous (t, hkv, d) per beam."""
    if ku is None:
        return 0, 0
    if ku.dim() != 5 or ku.stride(4) != 1 or ku.stride(3) != ku.shape[4] or ku.stride(2) != ku.shape[3] * ku.shape[4]:
        raise ValueError("unshared k/v must be [n_req][bw][nd][hkv][d] with contiguous (nd, hkv, d)")
    return ku.stride(0), ku.stride(1)


def attn_staged(q, ks, vs, ku, vu, n_unshared, hkv, scale, out=None, lse=None, stream=None):
    """One decode step of staged attention (xgr_attn_staged): shared stage on the tensor cores,
    unshared stage + OnlineSoftmax merge in its epilogue. Returns the bf16 output
    [n_req][bw][hq][d] (and fills lse [n_req][bw][hq] fp32 if given)."""
    import torch
    n_req, bw, hq, d = _attn_shapes(q, ks)
    ls = 0 if ks is None else ks.shape[1]
    rs, bs = _unshared_strides(ku)
    if out is None:
        out = torch.empty_like(q)
    st = torch.cuda.current_stream() if stream is None else stream
    _check(lib.xgr_attn_staged(_ptr(q), _ptr(ks), _ptr(vs), ls, _ptr(ku), _ptr(vu), rs, bs, n_unshared,
                               _ptr(out), _ptr(lse), n_req, bw, hq, hkv, d, float(scale),
                               ctypes.c_void_p(st.cuda_stream)))
    return out


def attn_shared(q, ks, vs, hkv, scale, stream=None):
    """Shared stage partials (xgr_attn_shared): (m, s, o) fp32."""
    import torch
    n_req, bw, hq, d = _attn_shapes(q, ks)
    ls = 0 if ks is None else ks.shape[1]
    m = torch.empty((n_req, bw, hq), dtype=torch.float32, device=q.device)
    s = torch.empty_like(m)
    o = torch.empty((n_req, bw, hq, d), dtype=torch.float32, device=q.device)
    st = torch.cuda.current_stream() if stream is None else stream
    _check(lib.xgr_attn_shared(_ptr(q), _ptr(ks), _ptr(vs), ls, _ptr(m), _ptr(s), _ptr(o), n_req, bw, hq, hkv, d,
                               float(scale), ctypes.c_void_p(st.cuda_stream)))
    return m, s, o


def attn_unshared(q, ku, vu, n_unshared, hkv, scale, stream=None):
    """Unshared stage partials (xgr_attn_unshared): (m, s, o) fp32."""
    import torch
    n_req, bw, hq, d = _attn_shapes(q, None)
    rs, bs = _unshared_strides(ku)
    m = torch.empty((n_req, bw, hq), dtype=torch.float32, device=q.device)
    s = torch.empty_like(m)
    o = torch.empty((n_req, bw, hq, d), dtype=torch.float32, device=q.device)
    st = torch.cuda.current_stream() if stream is None else stream
    _check(lib.xgr_attn_unshared(_ptr(q), _ptr(ku), _ptr(vu), rs, bs, n_unshared, _ptr(m), _ptr(s), _ptr(o), n_req,
                                 bw, hq, hkv, d, float(scale), ctypes.c_void_p(st.cuda_stream)))
    return m, s, o


def attn_merge(p1, p2, with_lse=False, stream=None):
    """OnlineSoftmax merge of two partials (xgr_attn_merge): returns out fp32 [..., d] (and lse)."""
    import torch
    m1, s1, o1 = p1
    m2, s2, o2 = p2
    d = o1.shape[-1]
    rows = m1.numel()
    out = torch.empty_like(o1)
    lse = torch.empty_like(m1) if with_lse else None
    st = torch.cuda.current_stream() if stream is None else stream
    _check(lib.xgr_attn_merge(_ptr(m1), _ptr(s1), _ptr(o1), _ptr(m2), _ptr(s2), _ptr(o2), rows, d, _ptr(out),
                              _ptr(lse), ctypes.c_void_p(st.cuda_stream)))
    return (out, lse) if with_lse else out


class ShardedBeamSearch:
    """One rank of a codebook-sharded beam search: wraps a BeamSearch with
    nranks > 1 and performs the two all-gathers between the shard phases.

    all_gather(t) -> tensor [nranks, *t.shape] in rank order. By default it is
    torch.distributed.all_gather_into_tensor on the given process group (NCCL over NVLink on a
    multi-GPU node); a single-process emulator passes its own concatenation."""

    def __init__(self, bs: "BeamSearch", group=None, all_gather=None):
        self.bs = bs
        self.group = group
        self._ag = all_gather or self._dist_all_gather

    def _dist_all_gather(self, t):
        import torch
        import torch.distributed as dist
        t = t.contiguous()
        out = torch.empty((self.bs.nranks * t.shape[0], *t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)   # concatenated along dim 0
        return out.view(self.bs.nranks, *t.shape)

    def step(self, logits_local, stream=None):
        """One decode step: two collectives (8 B per row of stats, 8 B per record)."""
        stats = self.bs.shard_stats(logits_local, stream)
        gstats = self._ag(stats)
        recs, _ = self.bs.shard_select(gstats, stream)
        grecs = self._ag(recs)
        self.bs.shard_merge(grecs, None, stream)

    def finalize(self, **kw):
        return self.bs.finalize(**kw)
