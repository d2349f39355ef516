"""Streams longer than 2^31 stages (64-bit stage and word indexing end to end):
one device decode of N = 2^31 + 12345 stages, checked against the oracle on
window-aligned sub-streams at the start, across the 2^31 boundary and at the
end.  A sub-stream starting at stage s0 = k*F reproduces the full stream's
windows k+1.. exactly (its window 0 lacks the left halo), up to its last
window, whose right halo is cut unless the sub-stream ends at N."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

K, GENS = 7, (0o171, 0o133)
F, V = 256, 42
N = (1 << 31) + 12345
SUB = 64 * F  # sub-stream length (a multiple of F)


@pytest.fixture(scope="module")
def stream():
    import torch
    g = torch.Generator(device="cuda").manual_seed(2011_13579)
    q = torch.empty((N, 2), dtype=torch.int8, device="cuda")
    q.random_(-128, 128, generator=g)
    return q


@pytest.fixture(scope="module", params=["16x2", "s32"])
def decoded(request, stream):
    import os

    import torch

    import paper_2011_13579_b200 as vt
    old = os.environ.get("VT_KERNEL_VARIANT")
    os.environ["VT_KERNEL_VARIANT"] = request.param
    try:
        words = vt.decode_stream_device(stream, vt.CodeSpec(K, GENS), F, V)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("VT_KERNEL_VARIANT", None)
        else:
            os.environ["VT_KERNEL_VARIANT"] = old
    return stream, words


def _bits(words, lo, hi):
    """Decoded bits [lo, hi) from the packed device words."""
    w0, w1 = lo // 32, -(-hi // 32)
    chunk = words[w0:w1].cpu().numpy().view(np.uint8)
    b = np.unpackbits(chunk, bitorder="little")
    return b[lo - 32 * w0: hi - 32 * w0]


@pytest.mark.parametrize("where", ["start", "boundary", "end"])
def test_stream_longer_than_2_31(decoded, where):
    q, words = decoded
    if where == "start":
        s0 = 0
    elif where == "boundary":
        s0 = ((1 << 31) // F - 32) * F  # the sub-stream straddles stage 2^31
    else:
        s0 = ((N - SUB) // F) * F
    s1 = N if where == "end" else s0 + SUB
    sub = q[s0:s1].cpu().numpy()
    want = oracle.decode_stream(sub, K, GENS, F, V, threads=8)
    # windows whose geometry matches the full stream's: all but the first (unless s0 = 0)
    # and the last (unless the sub-stream ends at N)
    lo = 0 if s0 == 0 else F
    hi = (s1 - s0) if s1 == N else (s1 - s0) - F
    got = _bits(words, s0 + lo, s0 + hi)
    np.testing.assert_array_equal(got, want[lo:hi])


@pytest.mark.parametrize("k,gens", [(9, (0o753, 0o561))], ids=["K9-multilane"])
def test_stream_longer_than_2_31_other_forms(stream, k, gens):
    """The multi-lane K=9 kernel on the same > 2^31-stage stream (the random int8 LLRs
    are as valid for (753,561) as for (171,133)): start, 2^31 boundary and end."""
    import torch

    import paper_2011_13579_b200 as vt
    words = vt.decode_stream_device(stream, vt.CodeSpec(k, gens), F, V)
    torch.cuda.synchronize()
    for s0, s1 in ((0, SUB), (((1 << 31) // F - 32) * F, ((1 << 31) // F - 32) * F + SUB),
                   (((N - SUB) // F) * F, N)):
        sub = stream[s0:s1].cpu().numpy()
        want = oracle.decode_stream(sub, k, gens, F, V, threads=8)
        lo = 0 if s0 == 0 else F
        hi = (s1 - s0) if s1 == N else (s1 - s0) - F
        np.testing.assert_array_equal(_bits(words, s0 + lo, s0 + hi), want[lo:hi])
