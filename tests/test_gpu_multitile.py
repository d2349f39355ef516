"""Launches in which every CTA decodes several tiles (window batches): the traceback
of tile i then runs interleaved with tile i+1's forward pass, one group step per
group end, and long windows (F = 1024) stress the traceback's 64-bit bit
accumulator between word flushes.  Each kernel form, V = 0 frames (independent
windows) checked against the oracle on the first and last 64 frames."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

# (K, generators, windows per CTA of the form, VT_KERNEL_VARIANT)
FORMS = [(7, (0o171, 0o133), 256, None), (7, (0o133, 0o171, 0o165), 256, None), (9, (0o753, 0o561), 64, None),
         (8, (0o247, 0o371), 64, None), (7, (0o171, 0o133), 128, "s32"), (9, (0o753, 0o561), 32, "s32"),
         (7, (0o171, 0o133), 256, "16x2tc"), (5, (0o23, 0o35), 128, None), (8, (0o247, 0o371), 64, "s32"),
         (7, (0o171, 0o133), 256, "16x2mma")]


@pytest.mark.parametrize("fl", [400, 1024])
@pytest.mark.parametrize("form", FORMS, ids=lambda f: f"K{f[0]}-{oct(f[1][0])}-{f[3] or 'default'}")
def test_multi_tile_long_windows(form, fl, monkeypatch):
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, variant = form
    if variant:
        monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    f = 2 * sms * wpc + 100  # > one tile per CTA at 2 CTAs per SM
    b = len(gens)
    q = np.random.default_rng(fl * 7 + k).integers(-128, 128, size=(f * fl, b)).astype(np.int8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), fl, 0)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=f * fl, bitorder="little").reshape(f, fl)
    sel = np.r_[0:64, f - 64:f]
    want, _ = oracle.decode_batch(np.transpose(q.reshape(f, fl, b)[sel], (0, 2, 1)), k, gens)
    np.testing.assert_array_equal(got[sel], want)


@pytest.mark.parametrize("form", FORMS[:4], ids=lambda f: f"K{f[0]}-{oct(f[1][0])}")
def test_multi_tile_overlapping_windows(form):
    """F = 256, V = 42 (the benchmark geometry) with several tiles per CTA: the
    oracle decodes window-aligned sub-streams at the start and the end (a
    sub-stream starting at stage k*F reproduces windows k+1.. exactly)."""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, _ = form
    F, V = 256, 42
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = (2 * sms * wpc + 300) * F + 77
    b = len(gens)
    q = np.random.default_rng(k * 11 + b).integers(-128, 128, size=(n, b)).astype(np.int8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), F, V)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    sub = 80 * F
    want = oracle.decode_stream(q[:sub], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[: sub - F], want[: sub - F])  # (the sub-stream's last window is cut)
    s0 = ((n - sub) // F) * F
    want = oracle.decode_stream(q[s0:], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[s0 + F:], want[F:])


@pytest.mark.parametrize("form", [FORMS[0], FORMS[2]], ids=["K7", "K9"])
def test_multi_tile_final_metrics(form):
    """decode_batch (final-metric kernels) with several tiles per CTA."""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, _ = form
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    f, fl = 2 * sms * wpc + 50, 100
    llrs = np.random.default_rng(k).integers(-128, 128, size=(f, len(gens), fl)).astype(np.int8)
    bits, metric = vt.decode_batch(llrs.astype(np.float64), vt.CodeSpec(k, gens))
    sel = np.r_[0:64, f - 64:f]
    wb, wm = oracle.decode_batch(llrs[sel], k, gens)
    np.testing.assert_array_equal(bits[sel], wb)
    np.testing.assert_array_equal(metric[sel], wm.astype(np.float64))


@pytest.mark.parametrize("form", [FORMS[0], FORMS[2]], ids=["K7", "K9"])
def test_multi_tile_window_range_pieces(form, tmp_path):
    """A long stream decoded as window-range pieces on stage sub-buffers (the file
    streaming / shard path, several tiles per CTA per piece) equals the whole decode."""
    import torch

    import paper_2011_13579_b200 as vt
    from paper_2011_13579_b200 import fileio
    k, gens, wpc, _ = form
    F, V = 256, 42
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 3 * (2 * sms * wpc + 100) * F + 5
    q = np.random.default_rng(k + 100).integers(-128, 128, size=(n, len(gens))).astype(np.int8)
    whole = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), F, V).cpu().numpy()
    p = tmp_path / "q.llr"
    fileio.write_llr_file(q.astype(np.float32).reshape(-1), str(p), "single")
    per = (2 * sms * wpc + 100)
    pieces = fileio.decode_llr_file(str(p), "single", vt.CodeSpec(k, gens), F, V, windows_per_piece=per)
    np.testing.assert_array_equal(pieces, whole)


@pytest.mark.parametrize("form", FORMS, ids=lambda f: f"K{f[0]}-{oct(f[1][0])}-{f[3] or 'default'}")
def test_multi_tile_deterministic(form, monkeypatch):
    """Repeated decodes of one multi-tile stream (uniform int8 LLRs: ties everywhere)
    return identical words.  (A history fetch issued right after the tile's last
    stores once returned stale data without the tile-end memory fence.)"""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, variant = form
    if variant:
        monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    F, V = 256, 42
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 3 * (2 * sms * wpc + 50) * F + 13
    q = torch.from_numpy(np.random.default_rng(99).integers(-128, 128, size=(n, len(gens))).astype(np.int8)).cuda()
    spec = vt.CodeSpec(k, gens)
    ref = vt.decode_stream_device(q, spec, F, V)
    for _ in range(5):
        assert int((vt.decode_stream_device(q, spec, F, V) != ref).sum().item()) == 0


@pytest.mark.parametrize("fv", [(200, 20), (100, 130), (33, 7)])
@pytest.mark.parametrize("form", [FORMS[0], FORMS[2], FORMS[4]], ids=["K7", "K9", "K7-s32"])
def test_multi_tile_unaligned_frames(form, fv, monkeypatch):
    """Frames that share output words with their neighbours (atomicOr merges), V > F,
    several tiles per CTA: deterministic and equal to the oracle on window-aligned
    sub-streams at both ends."""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, variant = form
    if variant:
        monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    F, V = fv
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = (2 * sms * wpc + 200) * F + 3
    q = np.random.default_rng(F + V + k).integers(-128, 128, size=(n, len(gens))).astype(np.int8)
    spec = vt.CodeSpec(k, gens)
    dq = torch.from_numpy(q).cuda()
    words = vt.decode_stream_device(dq, spec, F, V)
    assert int((vt.decode_stream_device(dq, spec, F, V) != words).sum().item()) == 0
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    m = max(2, -(-V // F) + 1)  # windows whose left halo is cut in a sub-stream starting at k*F
    sub = (m + 40) * F
    want = oracle.decode_stream(q[:sub], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[: sub - m * F], want[: sub - m * F])
    s0 = ((n - sub) // F) * F
    want = oracle.decode_stream(q[s0:], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[s0 + m * F:], want[m * F:])


@pytest.mark.parametrize("chunks", [1, 3])
def test_multi_tile_host_entry(chunks):
    """vt_decode_stream_host (pinned host buffers, pipelined pieces) with several tiles
    per CTA per piece equals the device-resident decode."""
    import torch

    import paper_2011_13579_b200 as vt
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    F, V = 256, 42
    n = 3 * (2 * sms * 256 + 100) * F + 9
    q = np.random.default_rng(chunks).integers(-128, 128, size=(n, 2)).astype(np.int8)
    spec = vt.default_spec()
    want = vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, F, V).cpu()
    got = vt.decode_stream_host(torch.from_numpy(q).pin_memory(), spec, F, V, nchunks=chunks)
    assert torch.equal(got, want)


def test_concurrent_threads_and_streams():
    """Decodes from several host threads, each on its own CUDA stream (device entry)
    or through the pipelined host entry, overlap on the GPU: each thread has its own
    scratch (per-stream workspace, per-thread staging) and gets the serial result."""
    import threading

    import torch

    import paper_2011_13579_b200 as vt
    spec = vt.default_spec()
    F, V = 256, 42
    rng = np.random.default_rng(1)
    streams_q = [rng.integers(-128, 128, size=(600_000 + 1000 * i, 2)).astype(np.int8) for i in range(4)]
    want = [vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, F, V).cpu() for q in streams_q]
    got = [None] * 8
    errors = []

    def work(i):
        try:
            q = streams_q[i % 4]
            if i < 4:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    dq = torch.from_numpy(q).cuda(non_blocking=False)
                    out = vt.decode_stream_device(dq, spec, F, V, stream=s)
                s.synchronize()
                got[i] = out.cpu()
            else:
                got[i] = vt.decode_stream_host(torch.from_numpy(q).pin_memory(), spec, F, V, nchunks=3).clone()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    for _ in range(3):
        threads = [threading.Thread(target=work, args=(i,)) for i in range(8)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors
        for i in range(8):
            assert torch.equal(got[i], want[i % 4]), i


def test_matrix_r4_optimized_large_batch():
    """decode_matrix_batch (radix-4 optimised tie order, thread-per-window kernel with
    several windows per thread) on a batch larger than the grid: every frame equals its
    own single-frame decode (per-thread scratch reused window after window)."""
    import torch

    import paper_2011_13579_b200 as vt
    spec = vt.default_spec()
    cfg = vt.DecoderConfig(radix=4, optimized=True)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    f, n = 2 * sms * 4 * 128 + 37, 61  # > 1 window per thread; odd length: final radix-2 step
    rng = np.random.default_rng(4)
    llrs = rng.integers(-8, 9, size=(f, 2, n)).astype(np.float64)  # tie-heavy
    res = vt.decode_matrix_batch(llrs, spec, cfg)
    for i in list(range(5)) + list(range(f - 5, f)) + [f // 2]:
        one = vt.decode_matrix_batch(llrs[i:i + 1], spec, cfg)
        np.testing.assert_array_equal(res.bits[i], one.bits[0])
        assert res.final_metric[i] == one.final_metric[0]


@pytest.mark.parametrize("form", [FORMS[0], FORMS[1], FORMS[2]], ids=["K7", "K7r3", "K9"])
def test_multi_tile_hard_decision_ties(form):
    """Hard-decision LLRs (+-1: ties at every stage) with several tiles per CTA:
    the tie rule holds at scale (oracle on window-aligned sub-streams)."""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, _ = form
    F, V = 256, 42
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = (2 * sms * wpc + 300) * F + 11
    q = (1 - 2 * np.random.default_rng(k + len(gens)).integers(0, 2, size=(n, len(gens)))).astype(np.int8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), F, V)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    sub = 60 * F
    want = oracle.decode_stream(q[:sub], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[: sub - F], want[: sub - F])
    s0 = ((n - sub) // F) * F
    want = oracle.decode_stream(q[s0:], k, gens, F, V, threads=8)
    np.testing.assert_array_equal(got[s0 + F:], want[F:])


@pytest.mark.parametrize("form", [FORMS[0], FORMS[2], FORMS[6], FORMS[1], FORMS[3]],
                         ids=["K7", "K9", "K7-tc", "K7r3", "K8"])
@pytest.mark.parametrize("tail", [130, 3])
def test_multi_tile_padding_skip_does_not_overrun_traceback(form, tail, monkeypatch):
    """V = 0 (no warm-up groups) with a short last window: a 16x2 thread decoding it
    would skip its leading zero padding, and in a CTA that decodes a tile after
    another tile its history stores could overtake that tile's traceback fetches
    (found by tools/stress_forms.py: whole windows garbled).  The host splits such a
    launch: the persistent grid over the windows before the hazardous suffix, one
    tile per CTA over the suffix (vt_capi.cu plan_launch)."""
    import torch

    import paper_2011_13579_b200 as vt
    k, gens, wpc, variant = form
    if variant:
        monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    F, V = 300, 0
    nw = 2 * sms * wpc + 16  # the last tile holds 16 windows, the last one `tail` stages long
    n = (nw - 1) * F + tail
    q = np.random.default_rng(k + tail).integers(-3, 4, size=(n, len(gens))).astype(np.int8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), F, V)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    for w in list(range(0, 2 * wpc, 7)) + list(range(nw - 40, nw)):
        s, e = w * F, min(n, (w + 1) * F)
        wb, _ = oracle.decode_batch(np.ascontiguousarray(q[s:e].T[None]), k, gens)
        np.testing.assert_array_equal(got[s:e], wb[0], err_msg=f"window {w}")


@pytest.mark.parametrize("form", [FORMS[0], FORMS[2]], ids=["K7", "K9"])
def test_hazard_split_keeps_workspace_capped(form):
    """The ragged-tail split costs one extra tile of scratch at most: the workspace of a
    V = 0 stream with a short last window stays within one CTA tile's slot of the
    aligned stream's (the earlier whole-launch fallback grew it with the window count)."""
    import paper_2011_13579_b200 as vt
    k, gens, wpc, _ = form
    spec = vt.CodeSpec(k, gens)
    F = 256
    for n in (1 << 24, 1 << 26):
        aligned = vt.workspace_bytes(spec, n, F, 0)
        ragged = vt.workspace_bytes(spec, n + 5, F, 0)
        assert ragged <= aligned * 1.01 + 4 * 1024 * 1024, (n, aligned, ragged)
