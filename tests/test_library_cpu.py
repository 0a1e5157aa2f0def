"""CPU-only checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol declared in include/*.h, and rejects bad arguments synchronously (before any
launch).  No compute call is made here (there is no GPU in this container)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2604_22312_b200 as gvr
    return gvr.library()


def _declared_functions():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            src = open(os.path.join(inc, fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", src, flags=re.M):
                name = m.group(1)
                if name not in ("if", "while", "defined"):
                    names.add(name)
    return names


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("gvr_topk_batched", "gvr_topk_batched_ex", "radix_topk_batched",
                     "radix_topk_batched_ex", "gvr_status_string", "gvr_topk_batched_host",
                     "gvr_workspace_create", "gvr_workspace_destroy", "gvr_version", "gvr_kernel_info"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_functions():
        assert hasattr(lib, name), f"{name} declared in include/ but not exported"


def test_sass_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2604_22312_b200",
                                                                  "libgvrtopk.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_status_strings(lib):
    assert lib.gvr_status_string(0) == b"GVR_OK"
    assert lib.gvr_status_string(1) == b"GVR_ERR_INVALID_ARGUMENT"
    assert lib.gvr_status_string(2) == b"GVR_ERR_UNSUPPORTED"
    assert lib.gvr_status_string(3) == b"GVR_ERR_CUDA"
    assert lib.gvr_status_string(99) == b"GVR_ERR_UNKNOWN"
    assert lib.gvr_version() >= 10000


def test_argument_validation_is_synchronous(lib):
    p = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first
    # k out of range
    assert lib.gvr_topk_batched(p, 10, None, 1, None, 0, p, None) == 1
    assert lib.gvr_topk_batched(p, 10, None, 1, None, 2049, p, None) == 2
    # negative rows / stride
    assert lib.gvr_topk_batched(p, 10, None, -1, None, 8, p, None) == 1
    assert lib.gvr_topk_batched(p, 0, None, 1, None, 8, p, None) == 1
    # null required pointers
    assert lib.gvr_topk_batched(None, 10, None, 1, None, 8, p, None) == 1
    assert lib.gvr_topk_batched(p, 10, None, 1, None, 8, None, None) == 1
    # stride too large for int32 indices
    assert lib.gvr_topk_batched(p, 1 << 31, None, 1, None, 8, p, None) == 2
    # partial overlap of prev and out
    assert lib.gvr_topk_batched(p, 10, None, 2, ctypes.c_void_p(0x1004), 8, p, None) == 1
    # zero rows is a no-op success (no launch)
    assert lib.gvr_topk_batched(None, 10, None, 0, None, 8, None, None) == 0
    assert lib.radix_topk_batched(p, 10, None, 1, 0, p, None) == 1
    assert lib.radix_topk_batched(None, 10, None, 0, 8, None, None) == 0
    # workspace argument checks
    h = ctypes.c_void_p()
    assert lib.gvr_workspace_create(0, 10, 8, ctypes.byref(h)) == 1
    assert lib.gvr_workspace_create(1, 10, 4096, ctypes.byref(h)) == 2
    assert lib.gvr_topk_batched_host(p, 10, None, 1, None, 8, p, None, None) == 1
    # CTA timeline diagnostic: unknown kernel id, or no output buffer when stopping
    assert lib.gvr_cta_timeline(2, 1, None, 0, None) == 1
    assert lib.gvr_cta_timeline(-1, 0, p, 4, None) == 1
    assert lib.gvr_cta_timeline(0, 0, None, 4, None) == 1
    assert lib.gvr_cta_timeline(1, 0, p, -1, None) == 1


def test_binding_fails_loudly_without_cuda():
    import torch
    import paper_2604_22312_b200 as gvr
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(gvr.GvrError):
        gvr.topk(torch.zeros(2, 100), 8)


def test_topk_host_validates_host_arrays():
    """topk_host checks its host arrays before the C call: a wrong-dtype or
    wrong-shape out is refused, row_lens / prev of another integer type are converted."""
    import types

    import numpy as np

    import paper_2604_22312_b200 as gvr
    ws = types.SimpleNamespace(k=2048, row_stride=16, max_rows=2, _h=None)
    s = np.zeros((2, 16), np.float32)
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(s, ws, 2048, out=np.zeros((2, 2048), np.int64))
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(s, ws, 2048, out=np.zeros((2, 1024), np.int32))
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(s, ws, 2048, row_lens=np.zeros(3, np.int64))
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(s, ws, 2048, prev=np.zeros((2, 7), np.int32))
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(np.zeros((3, 16), np.float32), ws, 2048)  # more rows than the workspace
    with pytest.raises(gvr.GvrError):
        gvr.topk_host(s.astype(np.float64), ws, 2048)
