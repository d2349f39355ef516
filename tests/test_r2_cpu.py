"""CPU checks for the round-2 additions: the oracle and the host-side code tables
against vectors the reference itself produced (tests/golden/make_golden_r2.py),
encode_batch against the reference's encode vectors, the C ABI's shard split
against sharding.shard_windows, and run-time code modules (jit.py) building and
registering without a GPU."""
import ctypes
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT, code_params, golden_cases

import paper_2011_13579_b200 as vt
from paper_2011_13579_b200 import _lib

GOLDEN_R2 = os.path.join(ROOT, "tests", "golden", "golden_r2.npz")


def _r2(kind):
    z = np.load(GOLDEN_R2)
    index = json.loads(bytes(z["index_json"]).decode())
    return [c for c in index["cases"] if c["kind"] == kind], index["codes"]


R2_STREAM, R2_CODES = _r2("stream")
R2_BATCH, _ = _r2("batch")
R2_DRAGONFLY, _ = _r2("dragonfly")
ENCODE, CODES = golden_cases("encode")


@pytest.fixture(scope="module")
def z2():
    return np.load(GOLDEN_R2)


@pytest.mark.parametrize("case", R2_STREAM, ids=[f"{c['code']}-{c['tag']}" for c in R2_STREAM])
def test_oracle_stream_matches_reference_for_other_codes(z2, case):
    k, gens = code_params(R2_CODES, case["code"])
    want = np.unpackbits(z2[case["key"] + "_bits"], count=case["n"], bitorder="little")
    got = oracle.decode_stream(z2[case["key"] + "_llr"], k, gens, case["frame_len"], case["overlap"], threads=2)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("case", R2_BATCH, ids=[c["code"] for c in R2_BATCH])
def test_oracle_batch_matches_reference_for_other_codes(z2, case):
    k, gens = code_params(R2_CODES, case["code"])
    bits, metric = oracle.decode_batch(z2[case["key"] + "_llr"], k, gens)
    np.testing.assert_array_equal(bits, z2[case["key"] + "_bits"])
    np.testing.assert_array_equal(metric.astype(np.float64), z2[case["key"] + "_metric"])


@pytest.mark.parametrize("case", R2_DRAGONFLY, ids=[f"{c['code']}-rho{c['rho']}" for c in R2_DRAGONFLY])
def test_dragonfly_tables_match_reference(z2, case):
    """compute_bomat / identical_bomat_classes / find_dragonfly_groups (codes.py:351-412)
    for every built-in code, incl. K=8/9 where the radix-4 optimisation is ineffective."""
    k, gens = code_params(R2_CODES, case["code"])
    spec = vt.CodeSpec(k, gens)
    rho = case["rho"]
    bomats = np.stack([vt.codes.compute_bomat(f, rho, spec) for f in range(spec.num_dragonflies(rho))])
    np.testing.assert_array_equal(bomats, z2[case["key"] + "_bomats"])
    assert [list(c) for c in vt.codes.identical_bomat_classes(rho, spec)] == case["classes"]
    groups = [{"representative": g.representative, "members": list(g.members),
               "permutations": {str(f): list(p) for f, p in g.permutations.items()}}
              for g in vt.codes.find_dragonfly_groups(rho, spec)]
    assert groups == case["groups"]


def test_radix4_optimisation_effective_flag_matches_reference():
    """Whether the dragonfly grouping beats the plain classes (pack_radix4's
    optimization_effective, matrix.py:206-220): K=7 and K=8 (247,371) group, K=9 and
    K=5 (23,35) fall back -- the flag that selects the permuted tie order."""
    from paper_2011_13579_b200.decoder import _radix4_tiles
    seen = 0
    for case in R2_DRAGONFLY:
        if case["rho"] != 2 or case["r4_effective"] is None:
            continue
        k, gens = code_params(R2_CODES, case["code"])
        _, effective = _radix4_tiles(vt.CodeSpec(k, gens), True)
        assert effective == case["r4_effective"], case["code"]
        seen += 1
    assert seen >= 7


@pytest.mark.parametrize("case", ENCODE, ids=[c["code"] for c in ENCODE])
def test_encode_batch_matches_reference(case):
    """codes.encode_batch (codes.py:216-230) of the package (not the oracle) against
    the reference's own encoder output."""
    z = np.load(GOLDEN)
    k, gens = code_params(CODES, case["code"])
    spec = vt.CodeSpec(k, gens)
    bits = z[case["key"] + "_in"]
    np.testing.assert_array_equal(vt.encode_batch(bits, spec), z[case["key"] + "_out"])
    for f in range(min(3, bits.shape[0])):
        np.testing.assert_array_equal(vt.encode(bits[f], spec).reshape(-1, len(gens)), z[case["key"] + "_out"][f])


@pytest.mark.parametrize("n,f,v", [(1 << 28, 256, 42), (10_001, 100, 20), (3_001, 7, 5), (2_000, 48, 0),
                                   (5, 256, 42)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_c_shard_range_matches_shard_windows(n, f, v, world):
    out = (ctypes.c_int64 * 4)()
    for g in range(world):
        _lib.check(_lib.lib().vt_shard_range(n, f, v, world, g, out))
        sh = vt.sharding.shard_windows(n, f, v, world, g)
        assert tuple(out) == (sh.w0, sh.w1, sh.st0, sh.st1)


def test_workspace_host_covers_every_chunk():
    spec = vt.default_spec()
    code = _lib.VtCode.from_spec(spec)
    L = _lib.lib()
    n, f, v = 1 << 22, 256, 42
    nw = n // f
    whole = L.vt_workspace_bytes_host(ctypes.byref(code), n, f, v, 0, nw, 8)
    for i in range(8):
        assert L.vt_workspace_bytes(ctypes.byref(code), n, f, v, nw * i // 8, nw * (i + 1) // 8) <= whole


def test_code_module_builds_and_registers_without_gpu():
    """A code outside the built-in table: jit.build_module generates the same kernel forms
    as the build, nvcc compiles them for sm_100a, vt_load_code_module registers them."""
    from paper_2011_13579_b200 import jit
    spec = vt.CodeSpec(5, (0o25, 0o33, 0o37, 0o31))
    code = _lib.VtCode.from_spec(spec)
    jit.ensure(spec)
    assert _lib.lib().vt_code_supported(ctypes.byref(code)) == 1
    assert any("j5_25_33_37_31" in p for p in jit.loaded_modules())
    assert _lib.lib().vt_workspace_bytes(ctypes.byref(code), 100_000, 256, 42, 0, 391) > 0


def test_code_module_rejects_unsupported_geometry():
    from paper_2011_13579_b200 import jit
    with pytest.raises(ValueError):
        jit.build_module(10, (0o1001, 0o1777))
    with pytest.raises(ValueError):
        jit.build_module(5, (0o25, 0o33, 0o37, 0o31, 0o21))


def test_load_code_module_reports_bad_paths():
    assert _lib.lib().vt_load_code_module(b"/nonexistent/libx.so") == _lib.VT_EINVAL
    assert b"cannot load" in _lib.lib().vt_last_error()


def test_foreign_frame_plan_is_recognised_by_geometry():
    """A FramePlan built by the reference's plan_frames (its own Window class, a tuple of
    windows) takes the fused one-launch path: recognised by geometry, not class."""
    from dataclasses import dataclass

    from paper_2011_13579_b200.decoder import _closed_form_plan

    @dataclass(frozen=True)
    class ForeignWindow:
        start: int
        stop: int
        emit_start: int
        emit_stop: int

    @dataclass(frozen=True)
    class ForeignPlan:
        total_stages: int
        frame_len: int
        overlap: int
        windows: tuple

    def foreign(n, f, v):
        return ForeignPlan(n, f, v, tuple(ForeignWindow(w.start, w.stop, w.emit_start, w.emit_stop)
                                          for w in vt.plan_frames(n, f, v).windows))

    for n, f, v in ((1000, 256, 42), (5000, 33, 7), (17, 256, 64), (4096, 64, 0)):
        assert _closed_form_plan(foreign(n, f, v))
    bad = foreign(1000, 256, 42)
    ws = list(bad.windows)
    ws[1] = ForeignWindow(ws[1].start + 1, ws[1].stop, ws[1].emit_start, ws[1].emit_stop)
    assert not _closed_form_plan(ForeignPlan(1000, 256, 42, tuple(ws)))
    assert not _closed_form_plan(ForeignPlan(1000, 256, 42, tuple(ws[:-1])))


R2_TILE, _ = _r2("tile")


@pytest.mark.parametrize("case", R2_TILE[::4], ids=[f"{c['code']}-n{c['n']}-r{c['radix']}{'o' if c['optimized'] else ''}"
                                                    f"-{c['accumulator']}-{int(c['renormalize'])}" for c in R2_TILE[::4]])
def test_tile_tables_model_matches_reference(z2, case):
    """The host tile tables (tiles.py, pack_radix2/4 restated) in their per-lane
    mma.sync fragment form, run through a numpy model of vt_tiles.cu, reproduce the
    reference's decode_matrix_batch incl. accumulator="half" (binary16 rounding of every
    tile result, overflow to inf on long frames) and the tile-op counter."""
    import tile_model
    k, gens = code_params(R2_CODES, case["code"])
    spec = vt.CodeSpec(k, gens)
    bits, metric, ops = tile_model.decode(z2[case["key"] + "_llr"].astype(np.int64), spec, case["radix"],
                                          case["optimized"], case["accumulator"] == "half", case["renormalize"])
    np.testing.assert_array_equal(bits, z2[case["key"] + "_bits"])
    np.testing.assert_array_equal(metric, z2[case["key"] + "_metric"])
    assert ops == int(z2[case["key"] + "_counter"][0])


@pytest.mark.parametrize("lock", ["1", "2"])
def test_lockstep_generator_knob_emits_barriers(lock):
    """VT_NT16=256 + VT_LOCK16 (the measured-and-rejected warp-pair lockstep form)
    still generates: 256-thread launch bounds, the NT-scaled traceback ring addressing and one
    barrier per LLR chunk; the default (128 threads) has neither."""
    import subprocess
    import sys

    csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2011_13579_b200", "csrc")
    prog = ("import gen_kernels16 as g; k = g.Gen16('vtk16_k7r2', 7, (0o171, 0o133)); print(k.kernel())")
    env = dict(os.environ, VT_NT16="256", VT_LOCK16=lock)
    src = subprocess.run([sys.executable, "-c", prog], cwd=csrc, env=env, capture_output=True, text=True,
                         check=True).stdout
    assert "__launch_bounds__(256, 1)" in src and "((j & 48u) << 8)" in src
    assert ("bar.sync %0, 64;" in src) if lock == "1" else ("__syncthreads();  // VT_LOCK16=2" in src)
    env = {k: v for k, v in os.environ.items() if k not in ("VT_NT16", "VT_LOCK16")}
    src = subprocess.run([sys.executable, "-c", prog], cwd=csrc, env=env, capture_output=True, text=True,
                         check=True).stdout
    assert "__launch_bounds__(128, 1)" in src and "((j & 48u) << 7)" in src and "VT_LOCK16" not in src
