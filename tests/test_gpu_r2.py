"""GPU parity for the round-2 additions:

* codes the library was not built with (kernels generated + compiled at first use,
  jit.py) against vectors the reference decoded (tests/golden/golden_r2.npz) and
  against the oracle on larger streams;
* the multi-device host entry (vt_decode_stream_host_multi: one shard, host thread
  and stream per listed device -- here several streams on cuda:0) equals the
  single-device decode bit for bit;
* decode_stream with a reference-built (duck-typed) FramePlan takes the one-launch path;
* BER points against the reference's own run_point samples (exact pairing) and its
  error counts (Monte-Carlo confidence intervals).
"""
import ctypes
import json
import math
import os

import numpy as np
import pytest

import oracle
from conftest import ROOT, code_params, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

GOLDEN_R2 = os.path.join(ROOT, "tests", "golden", "golden_r2.npz")


def _r2(kind):
    z = np.load(GOLDEN_R2)
    index = json.loads(bytes(z["index_json"]).decode())
    return [c for c in index["cases"] if c["kind"] == kind], index["codes"]


R2_STREAM, R2_CODES = _r2("stream")
R2_BATCH, _ = _r2("batch")
R2_BER, _ = _r2("ber")


@pytest.fixture(scope="module")
def z2():
    return np.load(GOLDEN_R2)


@pytest.fixture(scope="module")
def vt():
    import paper_2011_13579_b200 as vt
    return vt


def _unpack(words, n):
    return np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")


@pytest.mark.parametrize("case", R2_STREAM, ids=[f"{c['code']}-{c['tag']}" for c in R2_STREAM])
def test_generated_code_stream_matches_reference(vt, z2, case):
    import torch
    k, gens = code_params(R2_CODES, case["code"])
    spec = vt.CodeSpec(k, gens)
    llr = z2[case["key"] + "_llr"]
    want = np.unpackbits(z2[case["key"] + "_bits"], count=case["n"], bitorder="little")
    words = vt.decode_stream_device(torch.from_numpy(llr).cuda(), spec, case["frame_len"], case["overlap"])
    np.testing.assert_array_equal(_unpack(words, case["n"]), want)
    plan = vt.plan_frames(case["n"], case["frame_len"], case["overlap"])
    np.testing.assert_array_equal(vt.decode_stream(llr.T.astype(np.float64), spec, plan), want)


@pytest.mark.parametrize("case", R2_BATCH, ids=[c["code"] for c in R2_BATCH])
def test_generated_code_batch_matches_reference(vt, z2, case):
    k, gens = code_params(R2_CODES, case["code"])
    bits, metric = vt.decode_batch(z2[case["key"] + "_llr"].astype(np.float64), vt.CodeSpec(k, gens))
    np.testing.assert_array_equal(bits, z2[case["key"] + "_bits"])
    np.testing.assert_array_equal(metric, z2[case["key"] + "_metric"])


@pytest.mark.parametrize("k,gens", [(7, (0o133, 0o171)), (5, (0o25, 0o33)), (5, (0o25, 0o33, 0o37, 0o31)),
                                    (9, (0o557, 0o663, 0o711)), (6, (0o65, 0o57)), (8, (0o345, 0o237)),
                                    (8, (0o237, 0o261, 0o313))])  # (K=8 B=3: the s32 form's shared memory goes dynamic)
@pytest.mark.parametrize("variant", [None, "s32"])
def test_generated_code_large_stream_vs_oracle(vt, k, gens, variant, monkeypatch):
    """Multi-tile launches of every generated form (16x2 / multi-lane 16x2 / s32) for
    codes outside the built-in table, against the oracle on window-aligned pieces."""
    import torch
    if variant:
        monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    spec = vt.CodeSpec(k, gens)
    n, f, v = 700_000 + 13, 256, 42
    _, q = oracle.synthetic_stream(n, k, gens, ebn0_db=1.5, seed=k * 100 + len(gens))
    got = _unpack(vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, f, v), n)
    sub = 40 * f
    want = oracle.decode_stream(q[:sub], k, gens, f, v, threads=8)
    np.testing.assert_array_equal(got[: sub - f], want[: sub - f])
    s0 = ((n - sub) // f) * f
    want = oracle.decode_stream(q[s0:], k, gens, f, v, threads=8)
    np.testing.assert_array_equal(got[s0 + f:], want[f:])


def test_generated_code_modules_are_in_tree(vt):
    from paper_2011_13579_b200 import jit
    vt.decode_batch(np.zeros((1, 2, 10)), vt.CodeSpec(6, (0o65, 0o57)))
    mods = jit.loaded_modules()
    assert mods and all(m.startswith(jit.JIT_DIR) for m in mods)


# ---------------------------------------------------------------------------
# multi-device host entry
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,f,v", [(1 << 22, 256, 42), (300_001, 100, 20), (50_003, 7, 5), (65_536, 48, 0),
                                   (1000, 256, 42)])
@pytest.mark.parametrize("devs", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0]])
def test_multi_device_entry_equals_single_device(vt, n, f, v, devs):
    import torch
    spec = vt.default_spec()
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=1.0, seed=n % 97)
    host = torch.from_numpy(q).pin_memory()
    single = vt.decode_stream_host(host, spec, f, v).clone()
    multi = vt.decode_stream_host(host, spec, f, v, devices=devs, nchunks=3)
    np.testing.assert_array_equal(multi.numpy(), single.numpy())
    np.testing.assert_array_equal(_unpack(single, n)[: 20 * f], oracle.decode_stream(q[: 22 * f + v], 7,
                                                                                      (0o171, 0o133), f, v)[: 20 * f])


def test_decode_stream_workers_fan_out(vt):
    """decode_stream(..., workers=G) (framing.py:121-135): up to G GPUs; same bits."""
    import torch
    spec = vt.default_spec()
    n = 200_000
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=2.0, seed=4)
    plan = vt.plan_frames(n, 256, 42)
    a = vt.decode_stream(q.T.astype(np.float64), spec, plan, workers=1)
    b = vt.decode_stream(q.T.astype(np.float64), spec, plan, workers=torch.cuda.device_count() + 3)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=8))


def test_multi_device_generated_code(vt):
    import torch
    spec = vt.CodeSpec(5, (0o25, 0o33, 0o37, 0o31))
    n = 123_457
    _, q = oracle.synthetic_stream(n, 5, spec.generators, ebn0_db=0.0, seed=9)
    host = torch.from_numpy(q).pin_memory()
    got = vt.decode_stream_host(host, spec, 256, 42, devices=[0, 0, 0], nchunks=2)
    np.testing.assert_array_equal(_unpack(got, n), oracle.decode_stream(q, 5, spec.generators, 256, 42, threads=8))


def test_multi_device_rejects_bad_devices(vt):
    import torch
    host = torch.zeros((1000, 2), dtype=torch.int8)
    with pytest.raises(ValueError):
        vt.decode_stream_host(host, vt.default_spec(), 256, 42, devices=[0, 99])


# ---------------------------------------------------------------------------
# reference-built plans, pinned staging reuse
# ---------------------------------------------------------------------------

def test_reference_shaped_plan_takes_the_fused_path(vt, monkeypatch):
    from dataclasses import dataclass

    from paper_2011_13579_b200 import decoder

    @dataclass(frozen=True)
    class W:
        start: int
        stop: int
        emit_start: int
        emit_stop: int

    @dataclass(frozen=True)
    class P:
        total_stages: int
        frame_len: int
        overlap: int
        windows: tuple

    n = 50_000
    _, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=2.0, seed=12)
    plan = P(n, 256, 42, tuple(W(w.start, w.stop, w.emit_start, w.emit_stop)
                               for w in vt.plan_frames(n, 256, 42).windows))

    def boom(*a, **k):
        raise AssertionError("took the per-length-group path")

    monkeypatch.setattr(decoder, "_decode_windows_general", boom)
    got = vt.decode_stream(q.T.astype(np.float64), vt.default_spec(), plan)
    np.testing.assert_array_equal(got, oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=8))
    got = vt.decode_stream(q.T.copy(), vt.default_spec(), plan)  # int8 input: the int path
    np.testing.assert_array_equal(got, oracle.decode_stream(q, 7, (0o171, 0o133), 256, 42, threads=8))


def test_repeated_host_decodes_reuse_pinned_staging(vt):
    spec = vt.default_spec()
    outs = []
    for seed in (1, 2, 1):
        _, q = oracle.synthetic_stream(30_000, 7, (0o171, 0o133), ebn0_db=2.0, seed=seed)
        outs.append(vt.decode_stream(q.T.astype(np.float64), spec, vt.plan_frames(30_000, 256, 42)))
    np.testing.assert_array_equal(outs[0], outs[2])  # results never alias the reused buffers
    assert not np.array_equal(outs[0], outs[1])
    vt.release_workspaces()


# ---------------------------------------------------------------------------
# BER against the reference's run_point
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", R2_BER, ids=[f"{c['ebn0_db']}dB" for c in R2_BER])
def test_ber_point_paired_with_reference_samples(vt, case):
    """rng="numpy" reproduces run_point's own samples (channel.py:113-136); on the int8
    quantisation the error count equals the reference decoder's exactly."""
    from paper_2011_13579_b200 import channel as ch
    p = ch.run_point(vt.default_spec(), case["ebn0_db"], case["n"], seed=case["seed"], frame_len=case["frame_len"],
                     point_index=case["point_index"], rng="numpy")
    assert (p.n, p.errors) == (case["n"], case["errors_int8"])


@pytest.mark.parametrize("case", R2_BER, ids=[f"{c['ebn0_db']}dB" for c in R2_BER])
def test_ber_point_gpu_rng_within_confidence_of_reference(vt, z2, case):
    """The fused GPU channel (independent Philox samples, 2^27 bits per point) agrees
    with the reference's int8 and float-LLR run_point counts within Monte-Carlo
    confidence: |z| < 4, with the variance of a point's BER taken from the reference's
    per-frame error counts (frames are independent; errors within a frame come in
    bursts: 3x to 18x the binomial variance from 4 dB down to 1 dB)."""
    from paper_2011_13579_b200 import channel as ch
    flen = case["frame_len"]
    g = ch.run_point(vt.default_spec(), case["ebn0_db"], 1 << 27, seed=123, frame_len=flen,
                     point_index=case["point_index"], rng="gpu")
    fe = z2[case["key"] + "_frame_errors"].astype(np.float64)
    var_frame = fe.var(ddof=1) / flen ** 2  # variance of one frame's BER
    n_ref_frames, n_gpu_frames = case["n"] // flen, g.n // flen
    s = math.sqrt(var_frame / n_ref_frames + var_frame / n_gpu_frames)
    for ref_err in (case["errors_int8"], case["errors_float"]):
        assert abs(g.errors / g.n - ref_err / case["n"]) < 4 * s + 1e-12, (case["ebn0_db"], ref_err, g)
