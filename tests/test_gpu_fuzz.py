"""Randomised geometry fuzz for the K=7 r1/2 kernel forms against the oracle:
stream length, frame length, overlap (incl. V > F, V = 0, F = 1, N < F), LLR
statistics (AWGN at several SNRs, saturated, uniform int8, sparse), and
window-range launches on stage sub-buffers, for every kernel form."""
import numpy as np
import pytest

from oracle import oracle

K, GENS = 7, (0o171, 0o133)
pytestmark = pytest.mark.gpu


def _cases(seed=20111357, count=24):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        f = int(rng.choice([1, 2, 5, 31, 32, 33, 64, 100, 255, 256, 257, 700, 4096]))
        v = int(rng.choice([0, 1, 7, 20, 42, 64, 130, 300]))
        n = int(rng.integers(1, 40_000))
        kind = ["awgn0", "awgn3", "awgn6", "saturated", "uniform", "sparse"][i % 6]
        out.append((n, f, v, kind, int(rng.integers(0, 1 << 30))))
    return out


def _llr(n, kind, seed):
    rng = np.random.default_rng(seed)
    if kind.startswith("awgn"):
        _, q = oracle.synthetic_stream(n, K, GENS, ebn0_db=float(kind[4:]), seed=seed & 0xFFFF, scale=16.0)
        return q
    if kind == "saturated":
        return rng.choice(np.array([-128, -127, 127], dtype=np.int8), size=(n, 2))
    if kind == "uniform":
        return rng.integers(-128, 128, size=(n, 2)).astype(np.int8)
    q = np.zeros((n, 2), dtype=np.int8)  # sparse: mostly zero (ties everywhere)
    m = rng.random((n, 2)) < 0.05
    q[m] = rng.integers(-128, 128, size=int(m.sum())).astype(np.int8)
    return q


@pytest.mark.parametrize("variant", ["16x2", "s32", "16x2tc", "16x2mma"])
@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"n{c[0]}-F{c[1]}-V{c[2]}-{c[3]}")
def test_fuzz_stream(case, variant, monkeypatch):
    import torch

    import paper_2011_13579_b200 as vt
    monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    n, f, v, kind, seed = case
    q = _llr(n, kind, seed)
    want = oracle.decode_stream(q, K, GENS, f, v, threads=8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(K, GENS), f, v)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("variant", ["16x2", "16x2tc", "16x2mma"])
@pytest.mark.parametrize("case", _cases(seed=7, count=6), ids=lambda c: f"n{c[0]}-F{c[1]}-V{c[2]}-{c[3]}")
def test_fuzz_window_ranges(case, variant, monkeypatch, tmp_path):
    """Window-range launches on stage sub-buffers (the streaming/sharding path)."""
    from paper_2011_13579_b200 import CodeSpec, fileio
    monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    n, f, v, kind, seed = case
    q = _llr(n, kind, seed)
    p = tmp_path / "q.llr"
    fileio.write_llr_file(q.astype(np.float64).reshape(-1), str(p), "single")
    per = max(1, (-(-n // f)) // 3)
    words = fileio.decode_llr_file(str(p), "single", CodeSpec(K, GENS), f, v, windows_per_piece=per)
    got = np.unpackbits(words.view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, oracle.decode_stream(q, K, GENS, f, v, threads=8))


# K=8 / K=9: the multi-lane 16x2 kernels (states over 2 / 4 lanes, shared-memory transpose,
# subset-minimum renormalisation) and the s32 kernels
_CODES89 = {"k9r2": (9, (0o753, 0o561)), "k8r2": (8, (0o247, 0o371))}


def _llr_code(n, kind, seed, k, gens):
    rng = np.random.default_rng(seed)
    if kind.startswith("awgn"):
        _, q = oracle.synthetic_stream(n, k, gens, ebn0_db=float(kind[4:]), seed=seed & 0xFFFF, scale=16.0)
        return q
    return _llr(n, kind, seed)


@pytest.mark.parametrize("variant", ["16x2", "s32"])
@pytest.mark.parametrize("code", sorted(_CODES89))
@pytest.mark.parametrize("case", _cases(seed=99, count=12), ids=lambda c: f"n{c[0]}-F{c[1]}-V{c[2]}-{c[3]}")
def test_fuzz_stream_k89(case, code, variant, monkeypatch):
    import torch

    import paper_2011_13579_b200 as vt
    monkeypatch.setenv("VT_KERNEL_VARIANT", variant)
    k, gens = _CODES89[code]
    n, f, v, kind, seed = case
    q = _llr_code(n, kind, seed, k, gens)
    want = oracle.decode_stream(q, k, gens, f, v, threads=8)
    words = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(k, gens), f, v)
    got = np.unpackbits(words.cpu().numpy().view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("case", _cases(seed=5, count=4), ids=lambda c: f"n{c[0]}-F{c[1]}-V{c[2]}-{c[3]}")
def test_fuzz_window_ranges_k9(case, tmp_path):
    """Window-range launches of the multi-lane kernel on stage sub-buffers."""
    from paper_2011_13579_b200 import CodeSpec, fileio
    k, gens = _CODES89["k9r2"]
    n, f, v, kind, seed = case
    q = _llr_code(n, kind, seed, k, gens)
    p = tmp_path / "q.llr"
    fileio.write_llr_file(q.astype(np.float64).reshape(-1), str(p), "single")
    per = max(1, (-(-n // f)) // 3)
    words = fileio.decode_llr_file(str(p), "single", CodeSpec(k, gens), f, v, windows_per_piece=per)
    got = np.unpackbits(words.view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, oracle.decode_stream(q, k, gens, f, v, threads=8))
