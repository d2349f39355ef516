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
         (7, (0o171, 0o133), 256, "16x2tc")]


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
