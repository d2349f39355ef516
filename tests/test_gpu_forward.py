"""reference.forward_batch / traceback_batch / forward / traceback and
decode_reference with non-uniform initial metrics on the GPU (csrc/vt_forward.cu)
against golden vectors from the unmodified reference
(tests/golden/make_forward_golden.py)."""
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
G = os.path.join(ROOT, "tests", "golden", "forward_golden.npz")
CODES = {"k3": (3, (0o7, 0o5)), "k7": (7, (0o171, 0o133)), "k7r3": (7, (0o133, 0o171, 0o165)),
         "k9": (9, (0o753, 0o561))}
TAGS = {"plain": {}, "renorm": {"renormalize": True}, "init": {"init": True},
        "init_renorm_hist": {"init": True, "renormalize": True, "keep_history": True}}


@pytest.fixture(scope="module")
def z():
    return np.load(G)


@pytest.mark.parametrize("tag", sorted(TAGS))
@pytest.mark.parametrize("name", sorted(CODES))
def test_forward_traceback_batch_match_reference(z, name, tag):
    from paper_2011_13579_b200 import CodeSpec, reference as R
    k, gens = CODES[name]
    spec = CodeSpec(k, gens)
    key = f"{name}_{tag}"
    kw = dict(TAGS[tag])
    if kw.pop("init", False):
        kw["initial_metrics"] = z[key + "_init"]
    surv, lam, hist = R.forward_batch(z[key + "_llr"].astype(np.float64), spec, **kw)
    np.testing.assert_array_equal(surv, z[key + "_surv"])
    np.testing.assert_array_equal(lam, z[key + "_lam"])
    if kw.get("keep_history"):
        np.testing.assert_array_equal(hist, z[key + "_hist"])
    else:
        assert hist is None
    np.testing.assert_array_equal(R.traceback_batch(surv, lam, spec), z[key + "_bits"])
    st = R.forward(z[key + "_llr"][1].astype(np.float64), spec, kw.get("initial_metrics"),
                   kw.get("renormalize", False))
    np.testing.assert_array_equal(R.traceback(st, spec), z[key + "_bits"][1])


@pytest.mark.parametrize("name", sorted(CODES))
def test_decode_reference_nonuniform_initial_metrics(z, name):
    import paper_2011_13579_b200 as vt
    k, gens = CODES[name]
    got = vt.decode_reference(z[f"{name}_decref_llr"].astype(np.float64), vt.CodeSpec(k, gens),
                              initial_metrics=z[f"{name}_decref_init"])
    np.testing.assert_array_equal(got, z[f"{name}_decref_bits"])


def test_forward_batch_rejects_fractional_inputs():
    from paper_2011_13579_b200 import CodeSpec, reference as R
    spec = CodeSpec(7, (0o171, 0o133))
    with pytest.raises(ValueError):
        R.forward_batch(np.full((1, 2, 5), 0.5), spec)
    with pytest.raises(ValueError):
        R.forward_batch(np.zeros((1, 2, 5)), spec, initial_metrics=np.full(64, 0.25))
