"""The paper's tile formulation on tensor cores (csrc/vt_tiles.cu, mma.sync.m16n8k16):
decode_matrix_batch against decode_matrix_batch results the reference produced --
radix 2, radix 4, radix 4 optimised, renormalised, the binary16 accumulator
(including frames whose binary16 metrics overflow to inf) -- and its tile-op counter
counted from the mma.sync the kernel issued."""
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT, code_params, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

GOLDEN_R2 = os.path.join(ROOT, "tests", "golden", "golden_r2.npz")
_Z = np.load(GOLDEN_R2)
_INDEX = json.loads(bytes(_Z["index_json"]).decode())
TILE = [c for c in _INDEX["cases"] if c["kind"] == "tile"]
CODES = _INDEX["codes"]


@pytest.mark.parametrize("case", TILE, ids=[f"{c['code']}-n{c['n']}-r{c['radix']}{'o' if c['optimized'] else ''}"
                                            f"-{c['accumulator']}-{int(c['renormalize'])}" for c in TILE])
def test_tile_decoder_matches_reference(case):
    import paper_2011_13579_b200 as vt
    k, gens = code_params(CODES, case["code"])
    cfg = vt.DecoderConfig(radix=case["radix"], optimized=case["optimized"], renormalize=case["renormalize"],
                           policy=vt.PrecisionPolicy(accumulator=case["accumulator"]))
    res = vt.decode_matrix_batch(_Z[case["key"] + "_llr"].astype(np.float64), vt.CodeSpec(k, gens), cfg)
    np.testing.assert_array_equal(res.bits, _Z[case["key"] + "_bits"])
    np.testing.assert_array_equal(res.final_metric, _Z[case["key"] + "_metric"])
    c = _Z[case["key"] + "_counter"]
    assert (res.counter.mma_ops, res.counter.survivor_write_passes, res.counter.stages) == tuple(int(x) for x in c)


def test_tile_counter_is_the_papers_q():
    """q = tile ops per stage: 2.0 radix-2, 0.5 radix-4 optimised for K=7 (PAPER.md:439,
    725; tests/test_matrix.py:148-156), counted from issued mma.sync."""
    import paper_2011_13579_b200 as vt
    spec = vt.default_spec()
    llr = np.random.default_rng(3).integers(-20, 21, size=(8, 2, 4096)).astype(np.float64)
    assert vt.decode_matrix_batch(llr, spec, vt.DecoderConfig(radix=2)).q == 2.0
    assert vt.decode_matrix_batch(llr, spec, vt.DecoderConfig(radix=4, optimized=True)).q == 0.5


def test_tile_decoder_large_batch_equals_fused_decoder():
    """On integer LLRs the single-precision tile decoder (radix 2 and radix 4
    unoptimised) equals the reference decoder: checked against the
    fused kernels on a large batch."""
    import paper_2011_13579_b200 as vt
    spec = vt.default_spec()
    llr = np.random.default_rng(5).integers(-128, 128, size=(3000, 2, 300)).astype(np.float64)
    bits, metric = vt.decode_batch(llr, spec)
    for radix in (2, 4):
        res = vt.decode_matrix_batch(llr, spec, vt.DecoderConfig(radix=radix))
        np.testing.assert_array_equal(res.bits, bits)
        np.testing.assert_array_equal(res.final_metric, metric)


def test_half_accumulator_ber_point_runs_on_tensor_cores():
    """run_point(decoder="matrix", accumulator="half") on the GPU channel: the binary16
    accumulator costs BER (the paper's C fp16 rows) but decodes."""
    import paper_2011_13579_b200 as vt
    from paper_2011_13579_b200 import channel as ch
    spec = vt.default_spec()
    half = vt.DecoderConfig(policy=vt.PrecisionPolicy(accumulator="half"))
    p_half = ch.run_point(spec, 3.0, 1 << 20, decoder="matrix", config=half, seed=4)
    p_single = ch.run_point(spec, 3.0, 1 << 20, decoder="matrix", seed=4)
    assert p_half.n == p_single.n == 1 << 20
    assert 0 < p_single.errors <= p_half.errors
    q = ch.run_point(spec, 3.0, 1 << 16, decoder="matrix", config=half, seed=4, rng="numpy")
    assert 0 < q.ber < 0.05 and math.isfinite(q.ber)
