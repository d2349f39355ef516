"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; API validation mirrors the reference's ValueErrors."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2011_13579_b200 as vt
from paper_2011_13579_b200 import _lib


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "vitertile_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(vt_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(L, s), s


def test_supported_codes_registry():
    L = _lib.lib()
    import ctypes
    for k, gens in ((7, (0o171, 0o133)), (7, (0o133, 0o171, 0o165)), (9, (0o753, 0o561)), (9, (0o561, 0o753)),
                    (3, (7, 5)), (8, (0o247, 0o371))):
        assert L.vt_code_supported(ctypes.byref(_lib.VtCode.from_spec(vt.CodeSpec(k, gens)))) == 1
    assert L.vt_code_supported(ctypes.byref(_lib.VtCode.from_spec(vt.CodeSpec(7, (0o155, 0o117))))) == 0


def test_plan_frames_matches_reference_examples():
    plan = vt.plan_frames(1000, frame_len=256, overlap=64)
    assert len(plan.windows) == 4
    w = plan.windows[1]
    assert (w.start, w.stop, w.emit_start, w.emit_stop) == (192, 576, 256, 512)
    assert plan.windows[-1].stop == 1000 and plan.windows[-1].start == 768 - 64
    with pytest.raises(ValueError):
        vt.plan_frames(0)
    with pytest.raises(ValueError):
        vt.plan_frames(10, frame_len=0)
    with pytest.raises(ValueError):
        vt.plan_frames(10, overlap=-1)
    big = vt.plan_frames(1 << 28, 256, 42)
    assert len(big.windows) == 1 << 20 and big.windows[-1].stop == 1 << 28


def test_codespec_validation_and_encode():
    with pytest.raises(ValueError):
        vt.CodeSpec(2, (3, 1))
    with pytest.raises(ValueError):
        vt.CodeSpec(7, (0o171,))
    with pytest.raises(ValueError):
        vt.CodeSpec(3, (0o17, 5))
    spec = vt.default_spec()
    assert spec.octal_generators == ("171", "133")
    assert vt.CodeSpec.from_octal(7, ["171", "133"]) == spec
    np.testing.assert_array_equal(vt.encode([1, 0, 0], spec)[:2], [1, 1])


def test_decode_argument_validation_without_gpu():
    spec = vt.default_spec()
    with pytest.raises(ValueError):
        vt.DecoderConfig(radix=3)
    with pytest.raises(ValueError):
        vt.PrecisionPolicy(accumulator="quarter")
    with pytest.raises(ValueError):
        vt.SoftFrame(np.zeros(4))
    with pytest.raises(ValueError):
        vt.decode_stream(np.zeros((2, 100)), spec, vt.plan_frames(200))
    with pytest.raises(ValueError):
        vt.decode_stream(np.zeros((2, 100)), spec, vt.plan_frames(100), decoder="magic")
    with pytest.raises(ValueError):  # non-integer LLRs must be quantised first
        vt.decode_batch(np.full((1, 2, 8), 0.5), spec)
    with pytest.raises(ValueError):
        vt.decode_batch(np.zeros((2, 3, 10)), spec)


def test_quantizer():
    q = vt.quantize_llr(np.array([0.01, -3.0, 100.0, -100.0]), scale=16)
    np.testing.assert_array_equal(q, np.array([0, -48, 127, -127], dtype=np.int8))


def test_pack_llr_f64_host_helper():
    """vt_pack_llr_f64 (host, no GPU): float64 (B, N) -> int8 (N, B) in one pass; rejects
    non-integers, NaN and out-of-range values with the lowest offending stage."""
    import ctypes
    L = _lib.lib()
    rng = np.random.default_rng(0)
    n = 300_001
    a = rng.integers(-128, 128, size=(3, n)).astype(np.float64)
    out = np.empty((n, 3), dtype=np.int8)
    vp = ctypes.c_void_p
    assert L.vt_pack_llr_f64(a.ctypes.data_as(vp), 3, n, n, out.ctypes.data_as(vp), 0) == 0
    np.testing.assert_array_equal(out, a.T.astype(np.int8))
    for bad, where in ((0.5, 200_000), (float("nan"), 77), (128.0, 5), (-129.0, 299_999), (float("inf"), 1)):
        b = a.copy()
        b[2, where] = bad
        assert L.vt_pack_llr_f64(b.ctypes.data_as(vp), 3, n, n, out.ctypes.data_as(vp), 4) == -1
        assert f"stage {where} " in L.vt_last_error().decode()


def test_pack_llr_f64_row_stride():
    """Rows of a wider buffer (row_stride > N): the (B, N) view of a (B, M) array."""
    import ctypes
    L = _lib.lib()
    a = np.random.default_rng(1).integers(-128, 128, size=(2, 1000)).astype(np.float64)
    out = np.empty((700, 2), dtype=np.int8)
    vp = ctypes.c_void_p
    assert L.vt_pack_llr_f64(a.ctypes.data_as(vp), 2, 700, 1000, out.ctypes.data_as(vp), 3) == 0
    np.testing.assert_array_equal(out, a[:, :700].T.astype(np.int8))
    assert L.vt_pack_llr_f64(a.ctypes.data_as(vp), 2, 700, 600, out.ctypes.data_as(vp), 3) == -1  # stride < N
