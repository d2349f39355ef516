"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle
from conftest import GOLDEN, code_params, golden_cases

STREAM, CODES = golden_cases("stream")
BATCH, _ = golden_cases("batch")
ENCODE, _ = golden_cases("encode")
CHANNEL, _ = golden_cases("channel")


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


@pytest.mark.parametrize("case", STREAM, ids=[f"{c['code']}-{c['tag']}" for c in STREAM])
def test_oracle_stream_matches_reference(z, case):
    k, gens = code_params(CODES, case["code"])
    llr = z[case["key"] + "_llr"]
    want = np.unpackbits(z[case["key"] + "_bits"], count=case["n"], bitorder="little")
    got = oracle.decode_stream(llr, k, gens, case["frame_len"], case["overlap"], threads=2)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("case", BATCH, ids=[f"{c['code']}-n{c['n']}-{c['mode']}-r{int(c['renormalize'])}"
                                              for c in BATCH])
def test_oracle_batch_matches_reference(z, case):
    k, gens = code_params(CODES, case["code"])
    bits, metric = oracle.decode_batch(z[case["key"] + "_llr"], k, gens, mode=case["mode"],
                                       renormalize=case["renormalize"])
    np.testing.assert_array_equal(bits, z[case["key"] + "_bits"])
    np.testing.assert_array_equal(metric.astype(np.float64), z[case["key"] + "_metric"])


@pytest.mark.parametrize("case", ENCODE, ids=[c["code"] for c in ENCODE])
def test_oracle_encode_matches_reference(z, case):
    k, gens = code_params(CODES, case["code"])
    np.testing.assert_array_equal(oracle.encode_batch(z[case["key"] + "_in"], k, gens), z[case["key"] + "_out"])


def test_oracle_channel_sources_match_reference(z):
    case = CHANNEL[0]
    np.testing.assert_array_equal(oracle.generate_bits(1000, case["seed"], case["stream"]), z[case["key"] + "_bits"])
    y = oracle.modulate_awgn(z[case["key"] + "_coded"], case["ebn0"], case["rate"], case["mod_seed"],
                             case["mod_stream"])
    np.testing.assert_array_equal(y, z[case["key"] + "_y"])


def test_oracle_plan_windows_matches_reference_examples():
    # tests/test_framing.py:31-45 worked examples; SURVEY.md §7.2(5) probe
    assert oracle.plan_windows(100, 256, 64) == [(0, 100, 0, 100)]
    assert oracle.plan_windows(1000, 256, 42) == [(0, 298, 0, 256), (214, 554, 256, 512),
                                                  (470, 810, 512, 768), (726, 1000, 768, 1000)]


def test_oracle_threads_do_not_change_result():
    bits, q = oracle.synthetic_stream(20000, 7, (0o171, 0o133), ebn0_db=2.0, seed=3)
    a = oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=1)
    b = oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=4)
    np.testing.assert_array_equal(a, b)
    assert np.count_nonzero(a != bits) < 200
