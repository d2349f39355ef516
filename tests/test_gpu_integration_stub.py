"""INTEGRATION.md §2 as written: the numpy-only ctypes stub a reference maintainer
would add (vitertile/_b200.py) is extracted from the document and executed, with
dev_alloc = cudaMalloc through ctypes (no torch on this path), against the
reference's golden stream vectors."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, code_params, cuda_available, golden_cases

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

STREAM, CODES = golden_cases("stream")


def _stub_source() -> str:
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 2. C ABI binding inside the reference"):]
    m = re.search(r"```python\n(# vitertile/_b200.py.*?)```", sec, flags=re.S)
    assert m, "INTEGRATION.md §2 has no stub block"
    return m.group(1)


@pytest.fixture(scope="module")
def stub():
    os.environ["VITERTILE_B200_LIB"] = os.path.join(ROOT, "paper_2011_13579_b200", "libvitertile_b200.so")
    ns: dict = {}
    exec(compile(_stub_source(), "INTEGRATION.md#2", "exec"), ns)
    return ns


@pytest.fixture(scope="module")
def dev_alloc():
    path = "/usr/local/cuda/lib64/libcudart.so.12"
    cudart = ctypes.CDLL(path if os.path.exists(path) else "libcudart.so.12")
    cudart.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
    cudart.cudaFree.argtypes = [ctypes.c_void_p]
    ptrs = []

    def alloc(nbytes):
        p = ctypes.c_void_p()
        assert cudart.cudaMalloc(ctypes.byref(p), max(int(nbytes), 16)) == 0
        ptrs.append(p.value)
        return p.value

    yield alloc
    for p in ptrs:
        cudart.cudaFree(p)


@pytest.mark.parametrize("case", STREAM[::3], ids=[f"{c['code']}-{c['tag']}" for c in STREAM[::3]])
def test_integration_stub_decodes_golden_streams(stub, dev_alloc, case):
    import paper_2011_13579_b200 as vt  # (CodeSpec / plan_frames only: the stub is the decode path)
    z = np.load(GOLDEN)
    k, gens = code_params(CODES, case["code"])
    llr = z[case["key"] + "_llr"]
    want = np.unpackbits(z[case["key"] + "_bits"], count=case["n"], bitorder="little")
    plan = vt.plan_frames(case["n"], case["frame_len"], case["overlap"])
    got = stub["decode_stream_b200"](llr.T.astype(np.float64), vt.CodeSpec(k, gens), plan, dev_alloc)
    np.testing.assert_array_equal(got, want)


def test_integration_stub_reports_errors_as_value_error(stub, dev_alloc):
    from dataclasses import replace

    import paper_2011_13579_b200 as vt
    bad = replace(vt.plan_frames(100, 256, 42), frame_len=0)
    with pytest.raises(ValueError):
        stub["decode_stream_b200"](np.zeros((2, 100)), vt.CodeSpec(7, (0o171, 0o133)), bad, dev_alloc)
