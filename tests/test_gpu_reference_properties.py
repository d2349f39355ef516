"""The reference's own decoder properties (pkg/tests/test_reference.py:61-146,
TestDecoding) through the B200 API, with integer (int8-quantised) LLRs -- the
domain the B200 decoder is exact on (the reference tests use float LLRs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vt():
    import paper_2011_13579_b200 as vt
    return vt


@pytest.fixture(scope="module")
def spec171(vt):
    return vt.CodeSpec(7, (0o171, 0o133))


def _bpsk(coded, b):  # (N, B) coded bits -> (B, N) +-1
    return (1.0 - 2.0 * np.asarray(coded, dtype=np.float64)).reshape(-1, b).T


def test_noiseless_round_trip(vt, spec171):  # test_reference.py:62-66
    bits = np.random.default_rng(3).integers(0, 2, 200, dtype=np.uint8)
    llr = _bpsk(vt.encode(bits, spec171), 2)
    np.testing.assert_array_equal(vt.decode_reference(llr, spec171), bits)


def test_hard_mode_round_trip(vt, spec171):  # test_reference.py:68-...
    bits = np.random.default_rng(4).integers(0, 2, 120, dtype=np.uint8)
    coded = np.asarray(vt.encode(bits, spec171)).reshape(-1, 2).T
    np.testing.assert_array_equal(vt.decode_reference(coded, spec171, mode="hard"), bits)


def test_decode_batch_matches_single(vt, spec171):  # test_reference.py:99-106
    from paper_2011_13579_b200 import reference as R
    llrs = np.random.default_rng(7).integers(-40, 41, size=(5, 2, 80)).astype(np.float64)
    bits, metrics = vt.decode_batch(llrs, spec171)
    for i in range(5):
        np.testing.assert_array_equal(bits[i], vt.decode_reference(llrs[i], spec171))
        assert metrics[i] == R.forward(llrs[i], spec171).final_metrics.max()


def test_renormalize_keeps_decisions(vt, spec171):  # test_reference.py:108-113
    llrs = np.random.default_rng(8).integers(-40, 41, size=(3, 2, 150)).astype(np.float64)
    plain, _ = vt.decode_batch(llrs, spec171)
    renorm, _ = vt.decode_batch(llrs, spec171, renormalize=True)
    np.testing.assert_array_equal(plain, renorm)


def test_initial_metrics_bias_start_state(vt, spec171):  # test_reference.py:115-124
    rng = np.random.default_rng(9)
    bits = rng.integers(0, 2, 100, dtype=np.uint8)
    llr = np.clip(np.rint(16 * (_bpsk(vt.encode(bits, spec171), 2) + rng.normal(0, 1, size=(2, 100)))), -127, 127)
    init = np.full(spec171.num_states, -1_000_000.0)
    init[0] = 0.0
    biased = vt.decode_reference(llr, spec171, initial_metrics=init)
    free = vt.decode_reference(llr, spec171)
    assert np.count_nonzero(biased != bits) <= np.count_nonzero(free != bits)


@pytest.mark.parametrize("scale", [2, 3])
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_positive_scaling_invariance(vt, scale, seed):  # test_reference.py:126-134
    spec = vt.CodeSpec(5, (0o23, 0o35))
    llr = np.random.default_rng(seed).integers(-40, 41, size=(2, 40)).astype(np.float64)
    np.testing.assert_array_equal(vt.decode_reference(llr, spec), vt.decode_reference(scale * llr, spec))


def test_tie_rule_prefers_second_predecessor(spec171):  # test_reference.py:136-139
    from paper_2011_13579_b200 import reference as R
    assert R.forward(np.zeros((2, 6)), spec171).survivors.all()


def test_single_error_is_corrected(vt, spec171):  # test_reference.py:141-146
    bits = np.random.default_rng(10).integers(0, 2, 80, dtype=np.uint8)
    llr = _bpsk(vt.encode(bits, spec171), 2)
    llr[1, 37] *= -1.0
    np.testing.assert_array_equal(vt.decode_reference(llr, spec171), bits)
