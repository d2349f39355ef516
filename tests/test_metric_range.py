"""The 16x2 kernels keep path metrics in 16-bit halves; their range argument
(gen_kernels16.py, gen_kernels16m.py) bounds the metric spread by 256 * W, W
the code's maximum output-difference weight over K-1 stages.  (171,133)
renormalises by state 0 (span 2*Delta); the r1/3 (133,171,165) and K=9
(753,561) by the minimum over a small state set T (span Delta + 256 * W_T, round 2;
the exact minimum, span Delta, in round 1).  CPU: the bound's inputs and adversarial streams' spreads; GPU: those
streams decode exactly."""
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle

CODES = {"k7r2": (7, (0o171, 0o133), 11, 1500), "k7r3": (7, (0o133, 0o171, 0o165), 15, 2500),
         "k9r2": (9, (0o753, 0o561), 13, 2000)}


def _adv(name):
    return os.path.join(ROOT, "tests", "golden", f"adversarial_{name}.npz")


def _gen16():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import Gen16, spread_weight
    return spread_weight, Gen16


def test_spread_bound_inputs():
    spread_weight, Gen16 = _gen16()
    _, gens, w6, _ = CODES["k7r2"]
    assert spread_weight(7, gens) == w6
    g = Gen16("k7r2", 7, gens)
    assert g.cheap and not g.xmin and g.L == 3 and g.Sb == 256 * w6 + 512
    # Lambda stays below 2^13 inside a group: Sb' + Delta + 3 stages of growth
    assert g.Sb + 256 * w6 + 3 * 512 < (1 << 13)


def test_spread_bound_inputs_r13_exact_min():
    spread_weight, Gen16 = _gen16()
    _, gens, w6, _ = CODES["k7r3"]
    assert spread_weight(7, gens) == w6
    g = Gen16("k7r3", 7, gens)
    # renormalising by state 0 would need 2*Delta + 3*768 < 2^13 (false); by the exact
    # minimum (to 0), Delta + 3 stages of growth fits 3-bit groups
    assert 2 * 256 * w6 + 3 * 768 >= (1 << 13)
    assert g.xmin and not g.cheap and g.L == 3
    assert 256 * w6 + 3 * 768 < (1 << 13)
    # round 2: the minimum over a 6-state set T instead of all 64 (gen_kernels16.renorm_set):
    # within 256 * W_T of the exact minimum, so the span grows by Sb' = 256 * W_T
    assert len(g.rset) == 6 and g.Sb == 256 * _w_t(7, gens, g.rset) == 256 * 7
    assert g.Sb + 256 * w6 + 3 * 768 < (1 << 13)


def test_spread_bound_inputs_k9_multilane():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16m import Gen16M
    spread_weight, _ = _gen16()
    k, gens, w, _ = CODES["k9r2"]
    assert spread_weight(k, gens) == w
    g = Gen16M("k9r2", k, gens, 4)
    # state-0 renormalisation would need 2*Delta + 3*512 < 2^13: 8192, one short
    assert 2 * 256 * w + 3 * 512 == (1 << 13)
    assert g.xmin and g.L == 3 and g.Sb + 256 * w + 3 * 512 < (1 << 13)
    # round 2: per group end, the minimum over a 2-state set on one lane
    assert g.rsets and all(len(T) <= 2 for T, _, _ in g.rsets)
    lo = [g.top - g.L * (ge + 1) for ge in range(g.GPB)]
    for (T, wt, lane), l0 in zip(g.rsets, lo):
        assert wt == _w_t(k, gens, T) and 256 * wt <= g.Sb
        assert all(((x >> l0) & (g.T - 1)) == lane for x in T)  # all on the owner lane


def _w_t(K, gens, T):
    """W_T = max over states m of min_{t in T} w[t ^ m]: the subset minimum's bound."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import weight_table
    w = weight_table(K, gens)
    return max(min(w[t ^ m] for t in T) for m in range(1 << (K - 1)))


def test_weight_table_bounds_metric_differences():
    """|Lambda(s) - Lambda(s')| <= 256 * w[s ^ s'] at every stage of a random and an
    adversarial stream (the inequality the subset minimum rests on)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import weight_table
    for name in ("k7r3", "k9r2"):
        k, gens = CODES[name][:2]
        S = 1 << (k - 1)
        w = np.array(weight_table(k, gens))
        x = np.arange(S)
        bound = 256 * w[x[:, None] ^ x[None, :]]
        rng = np.random.default_rng(5)
        for q in (np.load(_adv(name))["llr"][:1500].astype(np.int64),
                  rng.integers(-128, 128, size=(1500, len(gens)))):
            m = _forward_metrics(q, k, gens)
            for t in range(0, len(m), 7):
                assert np.all(np.abs(m[t][:, None] - m[t][None, :]) <= bound)


def _forward_metrics(q, k, gens):
    S = 1 << (k - 1)

    def par(x):
        return bin(x).count("1") & 1
    p0 = np.array([2 * (j % (S // 2)) for j in range(S)])
    sg0 = np.array([[1 - 2 * par(g & ((j >> (k - 2)) << (k - 1) | p0[j])) for g in gens] for j in range(S)])
    sg1 = np.array([[1 - 2 * par(g & ((j >> (k - 2)) << (k - 1) | (p0[j] + 1))) for g in gens] for j in range(S)])
    m = np.zeros(S, np.int64)
    out = []
    for t in range(q.shape[0]):
        m = np.maximum(m[p0] + sg0 @ q[t], m[p0 + 1] + sg1 @ q[t])
        m -= m.min()
        out.append(m.copy())
    return out


@pytest.mark.parametrize("name", ["k7r3", "k9r2"])
def test_adversarial_gap_stream_within_bound(name):
    """The subset-minimum streams (make_adversarial_gap.py) push min_T Lambda - min Lambda
    up; it never exceeds the generator's Sb' = 256 * W_T."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import Gen16
    from gen_kernels16m import Gen16M
    k, gens = CODES[name][:2]
    g = Gen16M(name, k, gens, 4) if k == 9 else Gen16(name, k, gens)
    sets = [r[0] for r in g.rsets] if k == 9 else [g.rset]
    q = np.load(_adv("gap_" + name))["llr"].astype(np.int64)
    worst = max(int(m[T].min() - m.min()) for m in _forward_metrics(q, k, gens) for T in sets)
    assert worst <= g.Sb
    assert worst >= 1000  # the stream really pushes the gap (regenerate with make_adversarial_gap.py)


@pytest.mark.parametrize("name", sorted(CODES))
def test_adversarial_stream_spread_within_bound(name):
    k, gens, w6, floor = CODES[name]
    q = np.load(_adv(name))["llr"].astype(np.int64)
    assert q.shape[1] == len(gens)
    S = 1 << (k - 1)

    def par(x):
        return bin(x).count("1") & 1
    p0 = np.array([2 * (j % (S // 2)) for j in range(S)])
    sg0 = np.array([[1 - 2 * par(g & ((j >> (k - 2)) << (k - 1) | p0[j])) for g in gens] for j in range(S)])
    sg1 = np.array([[1 - 2 * par(g & ((j >> (k - 2)) << (k - 1) | (p0[j] + 1))) for g in gens] for j in range(S)])
    m = np.zeros(S, np.int64)
    worst = 0
    for t in range(q.shape[0]):
        m = np.maximum(m[p0] + sg0 @ q[t], m[p0 + 1] + sg1 @ q[t])
        m -= m.max()
        worst = max(worst, -int(m.min()))
    assert worst <= 256 * w6
    assert worst >= floor  # the stream really is adversarial (regenerate with make_adversarial.py)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["k7r3", "k9r2"])
@pytest.mark.parametrize("fv", [(256, 42), (1000, 60), (31, 7), (24000, 0)])
def test_adversarial_gap_stream_decodes_exactly(name, fv):
    import paper_2011_13579_b200 as vt
    import torch
    k, gens = CODES[name][:2]
    q = np.load(_adv("gap_" + name))["llr"]
    f, v = fv
    want = oracle.decode_stream(q, k, gens, f, v, threads=8)
    out = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), f, v)
    got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=q.shape[0], bitorder="little")
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["16x2", "s32", "16x2mma"])
@pytest.mark.parametrize("name", sorted(CODES))
@pytest.mark.parametrize("fv", [(256, 42), (1000, 60), (31, 7), (24000, 0)])
def test_adversarial_stream_decodes_exactly(name, fv, variant, monkeypatch):
    import paper_2011_13579_b200 as vt
    import torch
    monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    k, gens = CODES[name][:2]
    q = np.load(_adv(name))["llr"]
    f, v = fv
    want = oracle.decode_stream(q, k, gens, f, v, threads=8)
    out = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), f, v)
    got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=q.shape[0], bitorder="little")
    np.testing.assert_array_equal(got, want)


def test_traceback_accumulator_capacity():
    """TracebackLite keeps < 32 unwritten bits after a settle in a 64-bit accumulator
    and gains L bits per traceback step; the 16x2 kernels settle once per LLR chunk
    (CHB bodies x GPB steps), so a chunk may add at most 33 bits unless the generator
    emits a mid-chunk settle."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
    from gen_kernels16 import Gen16
    from gen_kernels16m import Gen16M
    gens = [Gen16("k7r2", 7, (0o171, 0o133)), Gen16("k7r3", 7, (0o133, 0o171, 0o165)),
            Gen16("k7r2", 7, (0o171, 0o133), tc=True), Gen16M("k9r2", 9, (0o753, 0o561), 4),
            Gen16M("k8r2", 8, (0o247, 0o371), 2)]
    for g in gens:
        per_chunk = g.CHB * g.GPB * g.L
        src = g.kernel()
        assert per_chunk <= 33 or "settle(a)" in src.split("it_start = 0;")[0], (g.name, per_chunk)
