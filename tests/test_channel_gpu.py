"""GPU BER harness: exact pairing with the reference's numpy streams, the
device channel's statistics, and BER-curve agreement with the reference's
published anchors (pkg/test_output.txt:19-23) within Monte-Carlo intervals."""
import math

import numpy as np
import pytest

import oracle
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def vt():
    import paper_2011_13579_b200 as vt
    return vt


def test_numpy_rng_point_is_exact_against_oracle(vt):
    from paper_2011_13579_b200 import channel as ch
    spec = vt.default_spec()
    p = ch.run_point(spec, 2.5, 200_000, seed=60, frame_len=1024, point_index=3, rng="numpy")
    # same frames through the oracle
    frames = -(-200_000 // 1024)
    data = ch.generate_bits(frames * 1024, 60, 3).reshape(frames, 1024)
    y = ch.modulate_awgn(vt.encode_batch(data, spec), ch.ChannelModel(2.5, seed=60), 0.5, 3)
    q = np.clip(np.rint(y * 16), -127, 127).astype(np.int8)
    bits, _ = oracle.decode_batch(np.transpose(q, (0, 2, 1)), 7, (0o171, 0o133))
    assert p.errors == int(np.count_nonzero(bits != data))
    assert p.n == frames * 1024


def test_gpu_channel_statistics_and_noiseless_decode(vt):
    import ctypes
    import torch
    from paper_2011_13579_b200 import _lib
    from paper_2011_13579_b200.decoder import _code, _ptr
    spec = vt.CodeSpec(7, (0o133, 0o171, 0o165))
    code = _code(spec)
    frames, flen = 64, 1000
    n = frames * flen
    bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    llr = torch.zeros(n * 3, dtype=torch.int8, device="cuda")
    sigma = 0.5
    _lib.check(_lib.lib().vt_channel_awgn(ctypes.byref(code), 5, 1, frames, flen, sigma, 16.0, 0, _ptr(bits),
                                          _ptr(llr), None))
    torch.cuda.synchronize()
    u = np.unpackbits(bits.cpu().numpy().view(np.uint8), count=n, bitorder="little").reshape(frames, flen)
    coded = vt.encode_batch(u, spec).reshape(n, 3)
    q = llr.cpu().numpy().reshape(n, 3).astype(np.float64)
    resid = q / 16.0 - (1.0 - 2.0 * coded)
    assert abs(u.mean() - 0.5) < 0.01
    assert abs(resid.mean()) < 0.01  # noise is zero-mean and the encoder matches codes.encode_batch
    assert abs(resid.std() - sigma) < 0.01
    # noiseless: the decode reproduces the source exactly
    _lib.check(_lib.lib().vt_channel_awgn(ctypes.byref(code), 5, 1, frames, flen, 0.0, 16.0, 0, _ptr(bits),
                                          _ptr(llr), None))
    torch.cuda.synchronize()
    u = np.unpackbits(bits.cpu().numpy().view(np.uint8), count=n, bitorder="little").reshape(frames, flen)
    dec, _ = vt.decode_batch(np.transpose(llr.cpu().numpy().reshape(frames, flen, 3), (0, 2, 1)).astype(float),
                             spec)
    np.testing.assert_array_equal(dec, u)


def test_gpu_rng_ber_agrees_with_numpy_rng(vt):
    from paper_2011_13579_b200 import channel as ch
    spec = vt.default_spec()
    a = ch.run_point(spec, 3.0, 2_000_000, seed=60, rng="numpy")
    b = ch.run_point(spec, 3.0, 50_000_000, seed=60, rng="gpu")
    # errors are bursty (~5 bits per error event): widen the binomial sigma accordingly
    s = math.sqrt(5 * (a.ber / a.n + b.ber / b.n))
    assert abs(a.ber - b.ber) < 4 * s, (a, b)


def test_soft_hard_gap_matches_reference_anchor(vt):
    """criterion 5 (tests/test_acceptance.py:156-168; test_output.txt:19):
    BER 1e-3 at 2.77 dB soft vs 4.92 dB hard (reference decoder on float LLRs)."""
    from paper_2011_13579_b200 import channel as ch
    spec = vt.default_spec()
    grid = [2.0 + 0.25 * i for i in range(15)]
    soft = ch.ber_sweep(spec, grid, 20_000_000, seed=50, mode="soft")
    hard = ch.ber_sweep(spec, grid, 20_000_000, seed=50, mode="hard")
    sx = ch.ebn0_at_ber([p for p in soft if p.valid], 1e-3)
    hx = ch.ebn0_at_ber([p for p in hard if p.valid], 1e-3)
    assert abs(sx - 2.77) < 0.12, sx
    assert abs(hx - 4.92) < 0.12, hx
    assert 1.5 <= hx - sx <= 2.5


def test_framing_penalty_matches_reference_anchor(vt):
    """criterion 7 (tests/test_acceptance.py:199-223; test_output.txt:23): errors over
    1e6 bits at 5 dB: unframed 0, F=256/V=64 0, V=0 89 -- same stream recipe,
    int8-quantised; GPU framed decodes equal the oracle on the same integers."""
    spec = vt.default_spec()
    n = 1_000_000
    rng = np.random.default_rng(70)
    bits = rng.integers(0, 2, n, dtype=np.uint8)
    coded = vt.encode(bits, spec).reshape(n, 2)
    y = 1.0 - 2.0 * coded + rng.normal(0.0, 1.0 / np.sqrt(10.0 ** 0.5), coded.shape)
    q = vt.quantize_llr(y, 16)
    framed = vt.decode_stream(q.T.astype(float), spec, vt.plan_frames(n, 256, 64))
    bare = vt.decode_stream(q.T.astype(float), spec, vt.plan_frames(n, 256, 0))
    np.testing.assert_array_equal(framed, oracle.decode_stream(q, 7, (0o171, 0o133), 256, 64, threads=8))
    np.testing.assert_array_equal(bare, oracle.decode_stream(q, 7, (0o171, 0o133), 256, 0, threads=8))
    e_framed, e_bare = int(np.count_nonzero(framed != bits)), int(np.count_nonzero(bare != bits))
    assert e_framed <= 3
    assert 89 - 4 * math.sqrt(89) <= e_bare <= 89 + 4 * math.sqrt(89), e_bare


@pytest.mark.parametrize("k,gens", [(7, (0o171, 0o133)), (9, (0o753, 0o561)), (3, (0o7, 0o5)),
                                    (7, (0o133, 0o171, 0o165))])
@pytest.mark.parametrize("flen", [37, 1023])
def test_gpu_encoder_matches_encode_batch_exactly(vt, k, gens, flen):
    """Noiseless channel: every LLR is +-16 exactly, i.e. the fused encoder equals
    codes.encode_batch (zero state at every frame start) for each code and frame length."""
    import ctypes
    import torch
    from paper_2011_13579_b200 import _lib
    from paper_2011_13579_b200.decoder import _code, _ptr
    spec = vt.CodeSpec(k, gens)
    b = len(gens)
    frames = 300
    n = frames * flen
    bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    llr = torch.zeros(((n * b + 15) // 16) * 16, dtype=torch.int8, device="cuda")
    _lib.check(_lib.lib().vt_channel_awgn(ctypes.byref(_code(spec)), 9, 2, frames, flen, 0.0, 16.0, 0, _ptr(bits),
                                          _ptr(llr), None))
    torch.cuda.synchronize()
    u = np.unpackbits(bits.cpu().numpy().view(np.uint8), count=n, bitorder="little").reshape(frames, flen)
    coded = vt.encode_batch(u, spec).reshape(n, b)
    q = llr.cpu().numpy()[: n * b].reshape(n, b)
    np.testing.assert_array_equal(q, (16 * (1 - 2 * coded.astype(np.int64))).astype(np.int8))


def test_matrix_decoder_points_use_the_radix4_tie_order(vt):
    """run_point(decoder="matrix", radix-4 optimised): both random sources decode with the
    dragonfly-permutation tie order (the numpy point equals decode_matrix_batch on the
    same quantised frames; the GPU point runs the r4perm kernel)."""
    from paper_2011_13579_b200 import channel as ch
    spec = vt.default_spec()
    cfg = vt.DecoderConfig(radix=4, optimized=True)
    p = ch.run_point(spec, 1.0, 50_000, decoder="matrix", config=cfg, seed=8, frame_len=500, point_index=2,
                     rng="numpy", llr_scale=2.0)  # coarse quantisation: ties
    frames = -(-50_000 // 500)
    data = ch.generate_bits(frames * 500, 8, 2).reshape(frames, 500)
    y = ch.modulate_awgn(vt.encode_batch(data, spec), ch.ChannelModel(1.0, seed=8), 0.5, 2)
    q = np.clip(np.rint(y * 2.0), -127, 127).astype(np.int8)
    bits = vt.decode_matrix_batch(np.transpose(q, (0, 2, 1)).astype(np.float32), spec, cfg).bits
    assert p.errors == int(np.count_nonzero(bits != data))
    g = ch.run_point(spec, 1.0, 200_000, decoder="matrix", config=cfg, seed=8, frame_len=500, point_index=2)
    r = ch.run_point(spec, 1.0, 200_000, seed=8, frame_len=500, point_index=2)
    assert g.n == r.n and abs(g.ber - r.ber) < 0.1 * r.ber  # same channel samples, different tie order
