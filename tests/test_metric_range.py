"""The 16x2 kernels keep path metrics in 16-bit halves; their range argument
(gen_kernels16.py) bounds the K=7 (171,133) metric spread by 256 * W6 with W6
the code's maximum output-difference weight over 6 stages.  CPU: the bound's
inputs and an adversarial stream's spread; GPU: that stream decodes exactly."""
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle

ADV = os.path.join(ROOT, "tests", "golden", "adversarial_k7r2.npz")
K, GENS = 7, (0o171, 0o133)


def _spread_weight():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import Gen16, spread_weight
    return spread_weight, Gen16


def test_spread_bound_inputs():
    spread_weight, Gen16 = _spread_weight()
    assert spread_weight(7, GENS) == 11
    g = Gen16("k7r2", 7, GENS)
    assert g.cheap and g.L == 3 and g.Sb == 256 * 11 + 512
    # Lambda stays below 2^13 inside a group: Sb' + Delta + 3 stages of growth
    assert g.Sb + 256 * 11 + 3 * 512 < (1 << 13)


def test_adversarial_stream_spread_within_bound():
    q = np.load(ADV)["llr"].astype(np.int64)
    S = 64

    def par(x):
        return bin(x).count("1") & 1
    p0 = np.array([2 * (j % 32) for j in range(S)])
    sg0 = np.array([[1 - 2 * par(g & ((j >> 5) << 6 | p0[j])) for g in GENS] for j in range(S)])
    sg1 = np.array([[1 - 2 * par(g & ((j >> 5) << 6 | (p0[j] + 1))) for g in GENS] for j in range(S)])
    m = np.zeros(S, np.int64)
    worst = 0
    for t in range(q.shape[0]):
        m = np.maximum(m[p0] + sg0 @ q[t], m[p0 + 1] + sg1 @ q[t])
        m -= m.max()
        worst = max(worst, -int(m.min()))
    assert worst <= 256 * 11
    assert worst >= 1500  # the stream really is adversarial (regenerate with make_adversarial.py)


@pytest.mark.gpu
@pytest.mark.parametrize("fv", [(256, 42), (1000, 60), (31, 7), (24000, 0)])
def test_adversarial_stream_decodes_exactly(fv):
    import paper_2011_13579_b200 as vt
    import torch
    q = np.load(ADV)["llr"]
    f, v = fv
    want = oracle.decode_stream(q, K, GENS, f, v, threads=8)
    out = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(K, GENS), f, v)
    got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=q.shape[0], bitorder="little")
    np.testing.assert_array_equal(got, want)
