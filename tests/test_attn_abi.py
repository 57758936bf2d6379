"""Host-side validation of the staged-attention C ABI (include/xgr_beam.h, xgr_attn_*): every
rejected call returns its status before any CUDA work, so these run without a GPU (not-gpu)."""
import ctypes

import pytest

XGR_ERR_INVALID_ARG, XGR_ERR_UNSUPPORTED, XGR_ERR_ALIGNMENT = 1, 2, 6
P = 0x10000   # a 16-byte aligned fake device address (never dereferenced: validation fails first)


def staged(**kw):
    from paper_2512_11529_b200 import binding
    a = dict(q=P, ks=P, vs=P, ls=64, ku=P, vu=P, rs=1024, bs=256, nu=2, out=P, lse=None,
             n_req=1, bw=4, hq=4, hkv=2, d=128, scale=0.088)
    a.update(kw)
    V = ctypes.c_void_p
    return binding.lib.xgr_attn_staged(V(a["q"]), V(a["ks"]), V(a["vs"]), a["ls"], V(a["ku"]), V(a["vu"]),
                                       a["rs"], a["bs"], a["nu"], V(a["out"]), V(a["lse"]), a["n_req"], a["bw"],
                                       a["hq"], a["hkv"], a["d"], ctypes.c_float(a["scale"]), None)


@pytest.mark.parametrize("kw,status", [
    (dict(d=64), XGR_ERR_UNSUPPORTED),            # head dim 128 only (DESIGN reading A4)
    (dict(hq=8, hkv=3), XGR_ERR_INVALID_ARG),     # hq % hkv != 0
    (dict(hq=12, hkv=4), XGR_ERR_UNSUPPORTED),    # G = 3 not a power of two
    (dict(ls=0, nu=0), XGR_ERR_INVALID_ARG),      # both stages empty
    (dict(nu=9), XGR_ERR_INVALID_ARG),            # more own tokens than ND <= 8
    (dict(bw=0), XGR_ERR_INVALID_ARG),
    (dict(scale=0.0), XGR_ERR_INVALID_ARG),
    (dict(q=P + 8), XGR_ERR_ALIGNMENT),
    (dict(ku=P + 4), XGR_ERR_ALIGNMENT),
    (dict(bs=100), XGR_ERR_ALIGNMENT),            # unshared strides: multiples of 8 elements
    (dict(out=None), XGR_ERR_INVALID_ARG),
    (dict(ks=None), XGR_ERR_INVALID_ARG),         # prompt tokens but no shared cache
])
def test_staged_rejects(kw, status):
    from paper_2512_11529_b200 import binding
    assert staged(**kw) == status
    assert binding.last_error()


def test_zero_requests_is_a_no_op():
    assert staged(n_req=0) == 0


def test_merge_and_partials_reject():
    from paper_2512_11529_b200 import binding
    V = ctypes.c_void_p
    lib = binding.lib
    assert lib.xgr_attn_merge(V(P), V(P), V(P), V(P), V(P), V(P), 10, 64, V(P), None, None) == XGR_ERR_UNSUPPORTED
    assert lib.xgr_attn_merge(V(P), V(P), V(P + 4), V(P), V(P), V(P), 10, 128, V(P), None, None) == XGR_ERR_ALIGNMENT
    assert lib.xgr_attn_merge(None, V(P), V(P), V(P), V(P), V(P), 10, 128, V(P), None, None) == XGR_ERR_INVALID_ARG
    assert lib.xgr_attn_shared(V(P), V(P), V(P), 64, None, V(P), V(P), 1, 4, 4, 2, 128, ctypes.c_float(0.1),
                               None) == XGR_ERR_INVALID_ARG
    assert lib.xgr_attn_unshared(V(P), V(P), V(P), 1024, 256, 2, V(P), V(P), V(P + 8), 1, 4, 4, 2, 128,
                                 ctypes.c_float(0.1), None) == XGR_ERR_ALIGNMENT
