"""CPU check of the 16x2 kernels' ALGORITHM (tests/kernel_model16.py mirrors the
generators' per-half arithmetic with 16-bit range assertions): against the
reference golden vectors and the oracle, including the adversarial
maximum-spread streams the range argument is tested with."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, code_params, golden_cases
from kernel_model16 import decode_stream_model16
from oracle import oracle

STREAM, CODES = golden_cases("stream")
CASES = [c for c in STREAM if c["code"] in ("k7r2", "k7r3", "k9r2") and c["n"] <= 20_000]


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


@pytest.mark.parametrize("case", CASES, ids=[f"{c['code']}-{c['tag']}" for c in CASES])
def test_model16_matches_reference(z, case):
    k, gens = code_params(CODES, case["code"])
    llr = z[case["key"] + "_llr"]
    want = np.unpackbits(z[case["key"] + "_bits"], count=case["n"], bitorder="little")
    np.testing.assert_array_equal(decode_stream_model16(llr, k, gens, case["frame_len"], case["overlap"]), want)


@pytest.mark.parametrize("name,k,gens", [("k7r2", 7, (0o171, 0o133)), ("k7r3", 7, (0o133, 0o171, 0o165)),
                                         ("k9r2", 9, (0o753, 0o561))])
def test_model16_adversarial_stream_in_range(name, k, gens):
    q = np.load(os.path.join(ROOT, "tests", "golden", f"adversarial_{name}.npz"))["llr"][:3000]
    want = oracle.decode_stream(q, k, gens, 256, 42, threads=4)
    np.testing.assert_array_equal(decode_stream_model16(q, k, gens, 256, 42), want)


@pytest.mark.parametrize("name,k,gens", [("k7r3", 7, (0o133, 0o171, 0o165)), ("k9r2", 9, (0o753, 0o561))])
def test_model16_adversarial_gap_stream_in_range(name, k, gens):
    q = np.load(os.path.join(ROOT, "tests", "golden", f"adversarial_gap_{name}.npz"))["llr"][:3000]
    want = oracle.decode_stream(q, k, gens, 256, 42, threads=4)
    np.testing.assert_array_equal(decode_stream_model16(q, k, gens, 256, 42), want)


def test_model16_range_check_has_teeth(monkeypatch):
    """With the renormalisation target below the spread bound (S_b' = 512 instead of
    Delta + 512) the adversarial stream drives a cheap-stage candidate negative."""
    import kernel_model16 as km
    real = km._gen

    def weak(K, gens):
        g = real(K, gens)
        g.Sb = 512
        return g
    monkeypatch.setattr(km, "_gen", weak)
    q = np.load(os.path.join(ROOT, "tests", "golden", "adversarial_k7r2.npz"))["llr"][:3000]
    with pytest.raises(AssertionError, match="16-bit half"):
        km.decode_stream_model16(q, 7, (0o171, 0o133), 256, 42)


@pytest.mark.parametrize("stream", ["adversarial_k7r2", "adversarial_gap_k7r2alt"])
def test_model16_alternating_form(stream, monkeypatch):
    """The alternating cheap/absorbing form (VT_ALT16): bit-exact and in range on the
    max-spread and subset-minimum-gap streams, and on the golden stream cases."""
    monkeypatch.setenv("VT_ALT16", "1")
    q = np.load(os.path.join(ROOT, "tests", "golden", f"{stream}.npz"))["llr"][:3000]
    gens = (0o171, 0o133)
    want = oracle.decode_stream(q, 7, gens, 256, 42, threads=4)
    np.testing.assert_array_equal(decode_stream_model16(q, 7, gens, 256, 42), want)


def test_model16_alternating_range_check_has_teeth(monkeypatch):
    """With the alternating form's renormalisation target at 0 instead of 256 * W_T + 2 * dmax
    the candidates leave the 16-bit half on the gap stream."""
    import kernel_model16 as km
    monkeypatch.setenv("VT_ALT16", "1")
    real = km._gen

    def weak(K, gens):
        g = real(K, gens)
        g.Sb_alt = 0
        return g
    monkeypatch.setattr(km, "_gen", weak)
    q = np.load(os.path.join(ROOT, "tests", "golden", "adversarial_gap_k7r2alt.npz"))["llr"][:3000]
    with pytest.raises(AssertionError, match="16-bit half"):
        km.decode_stream_model16(q, 7, (0o171, 0o133), 256, 42)
