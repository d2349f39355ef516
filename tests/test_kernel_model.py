"""CPU check of the kernel ALGORITHM (tests/kernel_model.py mirrors the
generated kernels' arithmetic) against the reference golden vectors."""
import numpy as np
import pytest

from conftest import GOLDEN, code_params, golden_cases
from kernel_model import decode_stream_model

STREAM, CODES = golden_cases("stream")
CASES = [c for c in STREAM if c["code"] in ("k7r2", "k7r3", "k5r2")]


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


@pytest.mark.parametrize("case", CASES, ids=[f"{c['code']}-{c['tag']}" for c in CASES])
def test_kernel_model_matches_reference(z, case):
    k, gens = code_params(CODES, case["code"])
    llr = z[case["key"] + "_llr"]
    want = np.unpackbits(z[case["key"] + "_bits"], count=case["n"], bitorder="little")
    np.testing.assert_array_equal(decode_stream_model(llr, k, gens, case["frame_len"], case["overlap"]), want)
