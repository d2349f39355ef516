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


# ---- framing (pkg/tests/test_framing.py:84-132) and matrix (test_matrix.py:136-211) ----

def _stream_llr(vt, spec, n, sigma, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, n, dtype=np.uint8)
    y = _bpsk(vt.encode(bits, spec), spec.outputs_per_bit) + sigma * rng.normal(size=(spec.outputs_per_bit, n))
    return bits, np.clip(np.rint(16 * y), -127, 127)


def test_framing_noiseless_equals_unframed(vt, spec171):
    bits, llr = _stream_llr(vt, spec171, 1500, 0.0, 23)
    np.testing.assert_array_equal(vt.decode_stream(llr, spec171, vt.plan_frames(1500, 256, 64)), bits)


@pytest.mark.parametrize("decoder,cfg", [("reference", None), ("matrix", dict(radix=2)),
                                         ("matrix", dict(radix=4, optimized=True))])
def test_framing_noisy_framed_close_to_unframed(vt, spec171, decoder, cfg):
    bits, llr = _stream_llr(vt, spec171, 3000, 0.7, 24)
    config = vt.DecoderConfig(**cfg) if cfg else None
    framed = vt.decode_stream(llr, spec171, vt.plan_frames(3000, 256, 64), decoder=decoder, config=config)
    unframed = vt.decode_reference(llr, spec171)
    assert np.count_nonzero(framed != bits) <= np.count_nonzero(unframed != bits) + 3


def test_framing_zero_overlap_is_worse_on_noisy_stream(vt, spec171):
    bits, llr = _stream_llr(vt, spec171, 20000, 0.85, 25)
    with_overlap = vt.decode_stream(llr, spec171, vt.plan_frames(20000, 256, 64))
    without = vt.decode_stream(llr, spec171, vt.plan_frames(20000, 256, 0))
    assert np.count_nonzero(without != bits) > np.count_nonzero(with_overlap != bits)


def test_framing_threaded_matches_serial(vt, spec171):
    _, llr = _stream_llr(vt, spec171, 4000, 0.9, 26)
    plan = vt.plan_frames(4000, 256, 64)
    np.testing.assert_array_equal(vt.decode_stream(llr, spec171, plan), vt.decode_stream(llr, spec171, plan, workers=4))


def test_framing_matrix_and_reference_agree_when_quiet(vt, spec171):
    _, llr = _stream_llr(vt, spec171, 2000, 0.3, 27)
    plan = vt.plan_frames(2000, 256, 64)
    ref = vt.decode_stream(llr, spec171, plan, decoder="reference")
    mat = vt.decode_stream(llr, spec171, plan, decoder="matrix", config=vt.DecoderConfig(radix=4, optimized=True))
    np.testing.assert_array_equal(ref, mat)


def test_framing_rejects_mismatched_plan_and_decoder(vt, spec171):
    _, llr = _stream_llr(vt, spec171, 100, 0.0, 28)
    with pytest.raises(ValueError):
        vt.decode_stream(llr, spec171, vt.plan_frames(200))
    with pytest.raises(ValueError):
        vt.decode_stream(llr, spec171, vt.plan_frames(100), decoder="magic")


@pytest.mark.parametrize("radix,optimized,q", [(2, False, 2.0), (4, False, 2.0), (4, True, 0.5)])
def test_matrix_noiseless_round_trip_and_ops(vt, spec171, radix, optimized, q):
    bits = np.random.default_rng(16).integers(0, 2, 128, dtype=np.uint8)
    llr = _bpsk(vt.encode(bits, spec171), 2)
    res = vt.decode_matrix(llr, spec171, vt.DecoderConfig(radix=radix, optimized=optimized))
    np.testing.assert_array_equal(res.bits, bits)
    assert res.q == q
    assert res.final_metric == 256.0


def test_matrix_tile_op_counts_per_length(vt, spec171):
    llrs = np.random.default_rng(17).integers(-20, 21, size=(2, 2, 11)).astype(np.float64)
    r2 = vt.decode_matrix_batch(llrs, spec171, vt.DecoderConfig(radix=2))
    assert r2.counter.mma_ops == 22 and r2.counter.survivor_write_passes == 11
    r4 = vt.decode_matrix_batch(llrs, spec171, vt.DecoderConfig(radix=4, optimized=True))
    assert r4.counter.mma_ops == 5 + 2 and r4.counter.survivor_write_passes == 6


@pytest.mark.parametrize("radix,optimized", [(2, False), (4, False), (4, True)])
def test_matrix_agrees_with_reference_on_noisy_frames(vt, spec171, radix, optimized):
    rng = np.random.default_rng(18)
    llrs = np.stack([_stream_llr(vt, spec171, 120, 0.9, 18 + i)[1] for i in range(6)])
    ref_bits, ref_metric = vt.decode_batch(llrs, spec171)
    res = vt.decode_matrix_batch(llrs, spec171, vt.DecoderConfig(radix=radix, optimized=optimized))
    np.testing.assert_array_equal(res.final_metric, ref_metric)  # exact in integers
    assert np.mean(res.bits != ref_bits) < 0.01


def test_matrix_renormalize_matches_plain(vt, spec171):
    llrs = np.stack([_stream_llr(vt, spec171, 90, 0.8, 19 + i)[1] for i in range(3)])
    plain = vt.decode_matrix_batch(llrs, spec171, vt.DecoderConfig(radix=4, optimized=True))
    renorm = vt.decode_matrix_batch(llrs, spec171, vt.DecoderConfig(radix=4, optimized=True, renormalize=True))
    np.testing.assert_array_equal(plain.bits, renorm.bits)
    np.testing.assert_array_equal(plain.final_metric, renorm.final_metric)


def test_matrix_rejects_bad_shapes_and_radix(vt, spec171):
    with pytest.raises(ValueError):
        vt.decode_matrix_batch(np.zeros((2, 3, 10)), spec171)
    with pytest.raises(ValueError):
        vt.DecoderConfig(radix=3)


@pytest.mark.parametrize("seed", range(6))
def test_matrix_radix_paths_agree_on_metric(vt, seed):
    spec = vt.CodeSpec(7, (0o171, 0o133))
    llrs = np.random.default_rng(seed).integers(-40, 41, size=(1, 2, 64)).astype(np.float64)
    metrics = [float(vt.decode_matrix_batch(llrs, spec, vt.DecoderConfig(radix=r, optimized=o)).final_metric[0])
               for r, o in ((2, False), (4, False), (4, True))]
    assert max(metrics) == min(metrics)
