"""The C-ABI library loads and exports every symbol include/xgr_beam.h declares; the ctypes
config struct matches the C layout; host-side validation answers without a GPU (not-gpu)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xgr_beam.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:xgr_status|const char\*|int32_t|int64_t)\s+(xgr_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2512_11529_b200 as xgr
    from paper_2512_11529_b200 import binding
    names = header_functions()
    assert len(names) >= 14
    assert sorted(binding.EXPORTS) == names
    for n in names:
        assert hasattr(xgr.lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", xgr.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    assert xgr.lib.xgr_abi_version() == binding.ABI_VERSION == 2
    # the ctypes mirror of xgr_config has the C layout (gcc: sizeof 104, dev_alloc at 56)
    assert ctypes.sizeof(binding.XgrConfig) == 104
    assert binding.XgrConfig.dev_alloc.offset == 56


def test_config_struct_layout_matches_c(tmp_path):
    from paper_2512_11529_b200.binding import XgrConfig
    c = tmp_path / "sz.c"
    c.write_text('#include "xgr_beam.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                 'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(xgr_config), offsetof(xgr_config, nccl_id),'
                 ' offsetof(xgr_config, flags), offsetof(xgr_config, dev_alloc), offsetof(xgr_config, dev_free),'
                 ' offsetof(xgr_config, alloc_user), offsetof(xgr_config, reserved));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(XgrConfig), XgrConfig.nccl_id.offset, XgrConfig.flags.offset,
                   XgrConfig.dev_alloc.offset, XgrConfig.dev_free.offset, XgrConfig.alloc_user.offset,
                   XgrConfig.reserved.offset]


def _cfg(**kw):
    from paper_2512_11529_b200.binding import XgrConfig
    c = XgrConfig()
    c.vocab, c.nd, c.beam_width, c.max_batch, c.nranks = 16, 3, 4, 1, 1
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("kw,status", [
    (dict(vocab=0), 1), (dict(vocab=65537), 1), (dict(nd=0), 1), (dict(nd=9), 1),
    (dict(beam_width=0), 1), (dict(beam_width=1025), 1), (dict(max_batch=0), 1),
    (dict(top_k=-1), 1), (dict(top_k=2, nranks=2, vocab=1024, beam_width=8), 2), (dict(nranks=2), 2), (dict(vocab=65536, nd=5), 2), (dict(flags=0x80), 1), (dict(reserved=(ctypes.c_int32 * 5)(1, 0, 0, 0, 0)), 1),
    (dict(dev_alloc="only_alloc"), 1), (dict(dev_free="only_free"), 1),
])
def test_init_validation_without_gpu(kw, status):
    from paper_2512_11529_b200 import binding
    # allocator hooks must come in pairs (checked before any CUDA call); these are never called
    if kw.get("dev_alloc") == "only_alloc":
        kw["dev_alloc"] = binding.DEV_ALLOC_FN(lambda n, u: None)
    if kw.get("dev_free") == "only_free":
        kw["dev_free"] = binding.DEV_FREE_FN(lambda p, u: None)
    h = ctypes.c_void_p()
    st = binding.lib.xgr_beam_init(ctypes.byref(_cfg(**kw)), ctypes.byref(h))
    assert st == status, binding.last_error()
    assert h.value is None
    assert binding.last_error()


def test_null_arguments():
    from paper_2512_11529_b200 import binding
    L = binding.lib
    assert L.xgr_beam_init(None, None) == 1
    assert L.xgr_mask_build(None, None, 0, None) == 1
    assert L.xgr_beam_step(None, 1, None, 1, 16, None) == 1
    assert L.xgr_beam_step_host(None, 1, None, 0, 1, 16, None) == 1
    assert L.xgr_beam_finalize(None, None, None, None, None, 0, None) == 1
    assert L.xgr_beam_destroy(None) == 0


def test_valid_config_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2512_11529_b200 import binding
    h = ctypes.c_void_p()
    st = binding.lib.xgr_beam_init(ctypes.byref(_cfg()), ctypes.byref(h))
    assert st == 8 and h.value is None
