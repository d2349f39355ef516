"""GPU parity: sm_100a decoder vs the reference (golden vectors) and vs the
C oracle on larger seeded inputs.  Bit-exact equality is required."""
import numpy as np
import pytest

import oracle
from conftest import GOLDEN, code_params, cuda_available, golden_cases

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

STREAM, CODES = golden_cases("stream")
BATCH, _ = golden_cases("batch")
MATRIX, _ = golden_cases("matrix")


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def vt():
    import paper_2011_13579_b200 as vt
    return vt


def _spec(vt, name):
    k, gens = code_params(CODES, name)
    return vt.CodeSpec(k, gens)


def _device_decode(vt, llr_nb, spec, f, v):
    import torch
    words = vt.decode_stream_device(torch.from_numpy(np.ascontiguousarray(llr_nb)).cuda(), spec, f, v)
    torch.cuda.synchronize()
    return np.unpackbits(words.cpu().numpy().view(np.uint8), count=llr_nb.shape[0], bitorder="little")


@pytest.mark.parametrize("case", STREAM, ids=[f"{c['code']}-{c['tag']}" for c in STREAM])
def test_stream_matches_reference_golden(vt, z, case):
    spec = _spec(vt, case["code"])
    llr = z[case["key"] + "_llr"]
    want = np.unpackbits(z[case["key"] + "_bits"], count=case["n"], bitorder="little")
    got = _device_decode(vt, llr, spec, case["frame_len"], case["overlap"])
    np.testing.assert_array_equal(got, want)
    # the reference-facing API (host (B, N) array in, uint8 bits out)
    plan = vt.plan_frames(case["n"], case["frame_len"], case["overlap"])
    np.testing.assert_array_equal(vt.decode_stream(llr.T.astype(np.float64), spec, plan), want)


@pytest.mark.parametrize("case", BATCH, ids=[f"{c['code']}-n{c['n']}-{c['mode']}-r{int(c['renormalize'])}"
                                              for c in BATCH])
def test_batch_matches_reference_golden(vt, z, case):
    spec = _spec(vt, case["code"])
    bits, metric = vt.decode_batch(z[case["key"] + "_llr"].astype(np.float64), spec, mode=case["mode"],
                                   renormalize=case["renormalize"])
    np.testing.assert_array_equal(bits, z[case["key"] + "_bits"])
    np.testing.assert_array_equal(metric, z[case["key"] + "_metric"])


@pytest.mark.parametrize("case", MATRIX, ids=[f"{c['code']}-n{c['n']}-r{c['radix']}{'o' if c['optimized'] else ''}"
                                               f"-{int(c['renormalize'])}" for c in MATRIX])
def test_matrix_matches_reference_golden(vt, z, case):
    spec = _spec(vt, case["code"])
    cfg = vt.DecoderConfig(radix=case["radix"], optimized=case["optimized"], renormalize=case["renormalize"])
    llr = z[case["key"] + "_llr"].astype(np.float64)
    res = vt.decode_matrix_batch(llr, spec, cfg)
    np.testing.assert_array_equal(res.bits, z[case["key"] + "_bits"])
    np.testing.assert_array_equal(res.final_metric, z[case["key"] + "_metric"])
    c = z[case["key"] + "_counter"]
    assert (res.counter.mma_ops, res.counter.survivor_write_passes, res.counter.stages) == tuple(int(x) for x in c)


def test_matrix_r4_optimized_stream_matches_reference_semantics(vt):
    """decode_stream(decoder="matrix", radix-4 optimised) on a noisy stream: windows are
    decoded independently, so it must equal decode_matrix_batch on each window."""
    spec = vt.default_spec()
    cfg = vt.DecoderConfig(radix=4, optimized=True)
    _, q = oracle.synthetic_stream(3000, 7, (0o171, 0o133), ebn0_db=1.0, seed=5, scale=4.0)  # tie-heavy
    plan = vt.plan_frames(3000, 256, 43)  # odd window lengths exercise the final radix-2 step
    got = vt.decode_stream(q.T.astype(float), spec, plan, decoder="matrix", config=cfg)
    want = np.zeros(3000, dtype=np.uint8)
    for w in plan.windows:
        bits = vt.decode_matrix_batch(q[w.start:w.stop].T[None].astype(float), spec, cfg).bits[0]
        want[w.emit_start:w.emit_stop] = bits[w.emit_start - w.start:w.emit_stop - w.start]
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("code", ["k7r2", "k7r3", "k9r2", "k8r2", "k5r2"])
@pytest.mark.parametrize("fv", [(256, 42), (64, 20), (1000, 100), (37, 5), (256, 0)])
def test_random_streams_match_oracle(vt, code, fv):
    k, gens = code_params(CODES, code)
    spec = vt.CodeSpec(k, gens)
    f, v = fv
    n = 60_000 if k <= 7 else 20_000
    _, q = oracle.synthetic_stream(n, k, gens, ebn0_db=1.5, seed=hash((code, fv)) & 0xFFFF, scale=20.0)
    want = oracle.decode_stream(q, k, gens, f, v, threads=8)
    np.testing.assert_array_equal(_device_decode(vt, q, spec, f, v), want)


def test_tie_heavy_and_extreme_llrs_match_oracle(vt):
    spec = vt.default_spec()
    rng = np.random.default_rng(5)
    for q in (rng.integers(-1, 2, size=(30_000, 2)).astype(np.int8),
              rng.choice(np.array([-128, 127], dtype=np.int8), size=(30_000, 2)),
              np.full((5000, 2), -128, dtype=np.int8)):
        want = oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=8)
        np.testing.assert_array_equal(_device_decode(vt, q, spec, 256, 42), want)


def test_window_ranges_on_sub_buffers_match_whole(vt):
    """vt_decode_stream_range on stage sub-buffers (the multi-GPU shard path)."""
    import ctypes
    import torch
    from paper_2011_13579_b200 import _lib
    from paper_2011_13579_b200.decoder import _code, _ptr, _workspace
    spec = vt.default_spec()
    n, f, v = 100_000, 256, 42
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=2.0, seed=17)
    whole = _device_decode(vt, q, spec, f, v)
    nw = -(-n // f)
    dev = torch.from_numpy(q).cuda()
    out = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    code = _code(spec)
    for w0, w1 in ((0, 100), (100, 101), (101, 250), (250, nw)):
        st0 = (max(0, w0 * f - v) // 16) * 16
        st1 = min(n, min(w1 * f, n) + v)
        sub = dev[st0:st1].clone()  # separate 16B-aligned allocation holding only the shard's stages
        need = _lib.lib().vt_workspace_bytes(ctypes.byref(code), n, f, v, w0, w1)
        ws = _workspace(need)
        _lib.check(_lib.lib().vt_decode_stream_range(ctypes.byref(code), _ptr(sub), st0, st1, n, f, v, w0, w1,
                                                     _ptr(out), None, _ptr(ws), ws.numel(), None))
    torch.cuda.synchronize()
    got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, whole)


def test_host_entry_matches_device_entry(vt):
    import torch
    spec = vt.default_spec()
    n = 200_003
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=2.5, seed=23)
    want = _device_decode(vt, q, spec, 256, 42)
    for chunks in (1, 3, 16):
        words = vt.decode_stream_host(torch.from_numpy(q).pin_memory(), spec, 256, 42, nchunks=chunks)
        got = np.unpackbits(words.numpy().view(np.uint8), count=n, bitorder="little")
        np.testing.assert_array_equal(got, want)


def test_final_metrics_match_oracle(vt):
    spec = vt.CodeSpec(7, (0o133, 0o171, 0o165))
    rng = np.random.default_rng(9)
    llrs = rng.integers(-128, 128, size=(300, 3, 500)).astype(np.int8)
    want_bits, want_metric = oracle.decode_batch(llrs, 7, (0o133, 0o171, 0o165))
    bits, metric = vt.decode_batch(llrs.astype(np.float64), spec)
    np.testing.assert_array_equal(bits, want_bits)
    np.testing.assert_array_equal(metric, want_metric.astype(np.float64))


@pytest.mark.parametrize("variant", ["16x2", "s32", "16x2tc", "16x2mma"])
@pytest.mark.parametrize("code", ["k7r2", "k7r3", "k8r2", "k9r2"])
@pytest.mark.parametrize("fv", [(256, 42), (100, 20), (37, 5)])
def test_kernel_variants_match_oracle(vt, code, fv, variant, monkeypatch):
    """Every kernel form is bit-exact (decoded bits and final metrics): the 16x2 kernels
    (two windows per thread; K=8/9 spread over 2/4 lanes), the one-window-per-thread s32
    kernels (VT_KERNEL_VARIANT=s32) and the tensor-core branch-metric form (K=7 r1/2)."""
    monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    k, gens = code_params(CODES, code)
    spec = vt.CodeSpec(k, gens)
    f, v = fv
    _, q = oracle.synthetic_stream(40_000, k, gens, ebn0_db=1.0, seed=11, scale=24.0)
    want = oracle.decode_stream(q, k, gens, f, v, threads=8)
    np.testing.assert_array_equal(_device_decode(vt, q, spec, f, v), want)
    bits, metric = vt.decode_batch(np.transpose(q[:30_000].reshape(60, 500, -1), (0, 2, 1)).astype(float), spec)
    wb, wm = oracle.decode_batch(np.transpose(q[:30_000].reshape(60, 500, -1), (0, 2, 1)), k, gens)
    np.testing.assert_array_equal(bits, wb)
    np.testing.assert_array_equal(metric, wm.astype(np.float64))


def test_device_entry_accepts_unaligned_slices(vt):
    """A row slice of an int8 (N, B) tensor starts at any byte; the entry re-aligns it."""
    import torch
    spec = vt.default_spec()
    _, q = oracle.synthetic_stream(20_001, 7, (0o171, 0o133), ebn0_db=2.0, seed=31)
    dq = torch.from_numpy(q).cuda()
    for off in (1, 3, 8):
        words = vt.decode_stream_device(dq[off:], spec, 256, 42)
        got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=q.shape[0] - off, bitorder="little")
        np.testing.assert_array_equal(got, oracle.decode_stream(q[off:], 7, (0o171, 0o133), 256, 42, threads=8))


def test_decode_stream_custom_window_plan(vt):
    """A FramePlan with a hand-built window list (not plan_frames' geometry) is decoded
    window by window like framing._decode_windows (grouped by length)."""
    from paper_2011_13579_b200.framing import FramePlan, Window
    spec = vt.default_spec()
    n = 5000
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=1.5, seed=41)
    cuts = [0, 700, 1500, 1600, 3333, 5000]
    wins = [Window(max(0, a - 50), min(n, b + 20), a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    plan = FramePlan(n, 1000, 50, wins)
    got = vt.decode_stream(q.T.astype(float), spec, plan)
    want = np.zeros(n, dtype=np.uint8)
    for w in wins:
        bits, _ = oracle.decode_batch(q[w.start:w.stop].T[None], 7, (0o171, 0o133))
        want[w.emit_start:w.emit_stop] = bits[0][w.emit_start - w.start:w.emit_stop - w.start]
    np.testing.assert_array_equal(got, want)
    got_m = vt.decode_stream(q.T.astype(float), spec, plan, decoder="matrix",
                             config=vt.DecoderConfig(radix=4, optimized=True))
    assert got_m.shape == (n,)


def test_decode_batch_large_float_batch_native_path(vt):
    """decode_batch on >= 2^20 float64 stages goes through the native pack helper
    (vt_pack_llr_f64 + a device transpose): same bits and metrics as the oracle;
    non-integer LLRs are rejected."""
    spec = vt.default_spec()
    rng = np.random.default_rng(12)
    llrs = rng.integers(-128, 128, size=(2100, 2, 500)).astype(np.float64)
    bits, metric = vt.decode_batch(llrs, spec)
    sel = np.r_[0:20, 2080:2100]
    wb, wm = oracle.decode_batch(llrs[sel].astype(np.int8), 7, (0o171, 0o133))
    np.testing.assert_array_equal(bits[sel], wb)
    np.testing.assert_array_equal(metric[sel], wm.astype(np.float64))
    llrs[1000, 1, 250] = 0.5
    with pytest.raises(ValueError):
        vt.decode_batch(llrs, spec)
