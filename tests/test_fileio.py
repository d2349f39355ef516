"""On-disk formats (cli.py:31-62) against files written by the reference's own
writers (tests/golden/make_fileio_golden.py), and the streaming file decoder /
``python -m paper_2011_13579_b200 decode`` against the oracle (GPU)."""
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle
from paper_2011_13579_b200 import CodeSpec, fileio

GOLD = os.path.join(ROOT, "tests", "golden", "fileio")
ARR = np.load(os.path.join(GOLD, "arrays.npz"))
K, GENS = 7, (0o171, 0o133)


@pytest.mark.parametrize("n", [0, 1, 13, 32, 33, 64, 1000])
def test_bit_file_byte_identical_to_reference_writer(tmp_path, n):
    bits = ARR[f"bits_{n}"]
    want = open(os.path.join(GOLD, f"bits_{n}.bin"), "rb").read()
    p = tmp_path / "b.bin"
    fileio.write_bit_file(bits, str(p))
    assert p.read_bytes() == want
    np.testing.assert_array_equal(fileio.read_bit_file(os.path.join(GOLD, f"bits_{n}.bin")), bits)
    # packed decoder words -> same bytes, no unpacking
    words = np.zeros((n + 31) // 32, dtype=np.int32)
    words.view(np.uint8)[: (n + 7) // 8] = np.packbits(bits, bitorder="little")
    words.view(np.uint8)[: (n + 7) // 8] |= 0  # (no stray bits beyond n by construction)
    q = tmp_path / "w.bin"
    fileio.write_packed_bit_file(words, n, str(q))
    assert q.read_bytes() == want


def test_packed_writer_masks_bits_beyond_count(tmp_path):
    words = np.array([-1], dtype=np.int32)  # all ones
    p = tmp_path / "w.bin"
    fileio.write_packed_bit_file(words, 5, str(p))
    want = tmp_path / "r.bin"
    fileio.write_bit_file(np.ones(5, np.uint8), str(want))
    assert p.read_bytes() == want.read_bytes()


@pytest.mark.parametrize("dtype", ["half", "single"])
@pytest.mark.parametrize("which", ["int", "float"])
def test_llr_file_matches_reference_writer(tmp_path, dtype, which):
    src = ARR[f"llr_{which}"]
    path = os.path.join(GOLD, f"llr_{which}_{dtype}.bin")
    p = tmp_path / "l.bin"
    fileio.write_llr_file(src, str(p), dtype)
    assert p.read_bytes() == open(path, "rb").read()
    got = fileio.read_llr_file(path, dtype)
    assert got.dtype == np.float64
    np.testing.assert_array_equal(got, src.astype("<f2" if dtype == "half" else "<f4").astype(np.float64))


def test_truncated_bit_file_raises(tmp_path):
    p = tmp_path / "t.bin"
    p.write_bytes(b"\x01\x02")
    with pytest.raises(ValueError):
        fileio.read_bit_file(str(p))
    p.write_bytes((100).to_bytes(8, "little") + b"\x00" * 4)
    with pytest.raises(ValueError):
        fileio.read_bit_file(str(p))


def test_bad_llr_dtype_raises(tmp_path):
    with pytest.raises(ValueError):
        fileio.write_llr_file(np.zeros(4), str(tmp_path / "x"), "double")


@pytest.mark.gpu
@pytest.mark.parametrize("fv,per", [((256, 42), 7), ((37, 5), 3), ((100, 64), 1000), ((1, 0), 50)])
@pytest.mark.parametrize("dtype", ["half", "single"])
def test_decode_llr_file_streams_pieces_exactly(tmp_path, fv, per, dtype):
    f, v = fv
    n = 20_000 if f > 1 else 3000
    _, q = oracle.synthetic_stream(n, K, GENS, ebn0_db=2.0, seed=9, scale=16.0)
    p = tmp_path / "s.llr"
    fileio.write_llr_file(q.astype(np.float64).reshape(-1), str(p), dtype)
    out = tmp_path / "s.out"
    words = fileio.decode_llr_file(str(p), dtype, CodeSpec(K, GENS), f, v, str(out) if n % 8 == 0 else None,
                                   windows_per_piece=per)
    want = oracle.decode_stream(q, K, GENS, f, v, threads=8)
    got = np.unpackbits(words.view(np.uint8), count=n, bitorder="little")
    np.testing.assert_array_equal(got, want)
    if n % 8 == 0:
        assert out.read_bytes() == np.packbits(want, bitorder="little").tobytes()


@pytest.mark.gpu
def test_cli_decode_matches_oracle(tmp_path):
    from paper_2011_13579_b200.__main__ import main
    n = 8192
    _, q = oracle.synthetic_stream(n, K, GENS, ebn0_db=2.5, seed=4, scale=16.0)
    llr = tmp_path / "in.llr"
    fileio.write_llr_file(q.astype(np.float64).reshape(-1), str(llr), "single")
    out = tmp_path / "out.bin"
    assert main(["decode", "--llr-in", str(llr), "--out", str(out), "--frame-len", "256", "--overlap", "42"]) == 0
    want = oracle.decode_stream(q, K, GENS, 256, 42, threads=8)
    assert out.read_bytes() == np.packbits(want, bitorder="little").tobytes()
    # coded-bit-file input (hard decisions, cli.py:141-145) through encode -> decode round trip
    data = np.random.default_rng(1).integers(0, 256, 64, dtype=np.uint8)
    raw = tmp_path / "data.bin"
    raw.write_bytes(data.tobytes())
    coded = tmp_path / "coded.bin"
    assert main(["encode", str(raw), "--out", str(coded)]) == 0
    dec = tmp_path / "dec.bin"
    assert main(["decode", str(coded), "--out", str(dec)]) == 0
    assert dec.read_bytes() == data.tobytes()  # noiseless: the decode recovers the data
