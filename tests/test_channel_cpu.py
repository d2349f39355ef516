"""BER-harness host logic (mirrors the reference's tests/test_channel.py
semantics) and the reference-exact numpy sources vs golden vectors."""
import math

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases
from paper_2011_13579_b200 import channel as ch

CHANNEL, _ = golden_cases("channel")


def test_sigma_conventions():
    m = ch.ChannelModel(3.0)
    assert m.sigma(0.5) == pytest.approx(math.sqrt(1.0 / (2 * 0.5 * 10 ** 0.3)))
    assert ch.ChannelModel(6.0, "shorthand").sigma(0.5) == pytest.approx(2 ** -0.3)
    with pytest.raises(ValueError):
        ch.ChannelModel(float("nan"))
    with pytest.raises(ValueError):
        ch.ChannelModel(1.0, "bogus")
    assert ch.ChannelModel(1.0).sigma(0.5) > ch.ChannelModel(2.0).sigma(0.5)


def test_numpy_sources_match_reference_golden():
    z = np.load(GOLDEN)
    case = CHANNEL[0]
    np.testing.assert_array_equal(ch.generate_bits(1000, case["seed"], case["stream"]), z[case["key"] + "_bits"])
    y = ch.modulate_awgn(z[case["key"] + "_coded"], ch.ChannelModel(case["ebn0"], seed=case["mod_seed"]),
                         case["rate"], stream=case["mod_stream"])
    np.testing.assert_array_equal(y, z[case["key"] + "_y"])
    with pytest.raises(ValueError):
        ch.generate_bits(0, 1)


def test_compute_ber_and_validity():
    p = ch.compute_ber(np.zeros(1000), np.r_[np.ones(5), np.zeros(995)], 3.0)
    assert (p.n, p.errors, p.ber, p.valid) == (1000, 5, 0.005, False)
    assert ch.compute_ber(np.zeros(10000), np.r_[np.ones(200), np.zeros(9800)]).valid
    with pytest.raises(ValueError):
        ch.compute_ber(np.zeros(3), np.zeros(4))


def test_ebn0_at_ber_interpolates():
    pts = [ch.BerPoint(1.0, 1000, 100, 0.1, True), ch.BerPoint(2.0, 1000, 10, 0.01, True)]
    assert ch.ebn0_at_ber(pts, 0.0316227766) == pytest.approx(1.5, abs=1e-6)
    with pytest.raises(ValueError):
        ch.ebn0_at_ber(pts, 1e-5)


def test_run_point_argument_validation():
    from paper_2011_13579_b200 import default_spec
    with pytest.raises(ValueError):
        ch.run_point(default_spec(), 3.0, 100, decoder="magic")
    with pytest.raises(ValueError):
        ch.run_point(default_spec(), 3.0, 100, mode="medium")


def test_csv(tmp_path):
    p = tmp_path / "ber.csv"
    ch.write_ber_csv([ch.BerPoint(3.0, 10, 1, 0.1, False)], str(p))
    assert p.read_text().splitlines()[1].startswith("3.0,10,1,0.1,0")


def test_csv_bytes_match_the_reference_writer(tmp_path):
    """Byte-identical to the reference's csv.writer rows (channel.py:168-173: CRLF
    dialect, ber formatted %.6g)."""
    import csv
    pts = [ch.BerPoint(2.5, 1000000, 1234, 0.001234, True), ch.BerPoint(3.0, 10, 1, 0.1, False),
           ch.BerPoint(0.25, 7, 0, 0.0, True)]
    want = tmp_path / "want.csv"
    with open(want, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["ebn0_db", "n", "errors", "ber", "valid"])
        for p in pts:
            w.writerow([p.ebn0_db, p.n, p.errors, f"{p.ber:.6g}", int(p.valid)])
    got = tmp_path / "got.csv"
    ch.write_ber_csv(pts, str(got))
    assert got.read_bytes() == want.read_bytes()


def test_ebn0_at_ber_first_crossing_and_flat_segment():
    pts = [ch.BerPoint(0.0, 10, 5, 0.5, True), ch.BerPoint(1.0, 10, 1, 0.1, True),
           ch.BerPoint(2.0, 10, 1, 0.1, True), ch.BerPoint(3.0, 10, 0, 0.0, True),
           ch.BerPoint(4.0, 100, 1, 0.01, True)]
    assert ch.ebn0_at_ber(pts, 0.1) == 1.0          # first bracketing pair, ber_lo == target
    assert ch.ebn0_at_ber(pts[1:3], 0.1) == 1.0     # flat segment
    # the 3.0 dB point has no errors: the crossing of 0.05 lies between 2.0 dB and 4.0 dB
    t = (np.log(0.1) - np.log(0.05)) / (np.log(0.1) - np.log(0.01))
    assert ch.ebn0_at_ber(pts, 0.05) == pytest.approx(2.0 + 2.0 * t, abs=1e-12)
