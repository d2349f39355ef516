"""gen_kernels16.renorm_set / weight_table (CPU): the subset-minimum renormalisation's
state sets.  The search must return a set T whose bound W_T = max_m min_{t in T} w[t ^ m]
is within the requested radius, of the smallest size (checked against brute force on
small codes), restricted to the allowed states, and the kernels' range conditions must
hold for every code the build compiles."""
import itertools
import os
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))
from gen_kernels16 import Gen16, renorm_set, spread_weight, weight_table  # noqa: E402


def _w_t(w, T, S):
    return max(min(w[t ^ m] for t in T) for m in range(S))


def test_weight_table_matches_spread_weight():
    for K, gens in ((5, (0o23, 0o35)), (7, (0o171, 0o133)), (7, (0o133, 0o171, 0o165)), (9, (0o753, 0o561))):
        w = weight_table(K, gens)
        assert len(w) == 1 << (K - 1) and w[0] == 0 and max(w) == spread_weight(K, gens)
        assert all(x > 0 for x in w[1:])  # a nonzero input difference always shows in the outputs


@pytest.mark.parametrize("K,gens", [(5, (0o23, 0o35)), (6, (0o53, 0o75)), (5, (0o27, 0o31, 0o35))])
def test_renorm_set_minimal_against_brute_force(K, gens):
    S = 1 << (K - 1)
    w = weight_table(K, gens)
    for wmax in range(0, max(w) + 1):
        r = renorm_set(K, gens, wmax)
        best = None
        for n in range(1, 4):
            for T in itertools.combinations(range(S), n):
                if _w_t(w, T, S) <= wmax:
                    best = n
                    break
            if best:
                break
        if best is None:  # no set of <= 3 states: the search may still find a larger one
            assert r is None or len(r[0]) > 3
            continue
        assert r is not None and len(r[0]) == best, (wmax, r, best)
        assert r[1] == _w_t(w, r[0], S) <= wmax


def test_renorm_set_respects_allowed_states():
    K, gens = 9, (0o753, 0o561)
    allowed = [s for s in range(256) if (s >> 3) & 3 == 0]
    T, wt = renorm_set(K, gens, 12, allowed=allowed)
    assert set(T) <= set(allowed) and wt <= 12


def test_compiled_codes_fit_the_16_bit_range():
    """Every 16x2 code the build compiles: the renormalisation target and the spread plus
    L stages of growth stay below 2^(16-L) (the generators assert the same)."""
    from gen_kernels import STANDARD_CODES
    from gen_kernels16m import Gen16M
    for name, (K, polys) in STANDARD_CODES.items():
        gens = tuple(int(p, 8) for p in polys)
        if K == 7:
            g = Gen16(name, K, gens)
        elif K in (8, 9):
            g = Gen16M(name, K, gens, {8: 2, 9: 4}[K])
        else:
            continue
        delta = 256 * spread_weight(K, gens)
        assert g.Sb + delta + g.L * 2 * g.dmax < (1 << (16 - g.L)), name
        if getattr(g, "rset", None):
            assert g.Sb == 256 * _w_t(weight_table(K, gens), g.rset, 1 << (K - 1))


def test_multilane_form_only_where_the_range_fits():
    """A K=9 code with four outputs spreads its metrics beyond 16-bit halves: its run-time
    module carries the s32 kernels alone (it used to assert in the generator)."""
    from gen_kernels import code_units
    from gen_kernels16m import Gen16M
    gens = (0o445, 0o605, 0o621, 0o713)
    assert not Gen16M("x", 9, gens, 4).supported
    assert [u[0] for u in code_units("x", 9, gens)] == ["vtk_x.cu"]
    assert Gen16M("x", 9, (0o557, 0o663, 0o711), 4).supported
