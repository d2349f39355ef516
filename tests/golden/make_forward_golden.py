"""Golden vectors for reference.forward_batch / traceback_batch / decode_reference
with non-uniform initial metrics, produced by the UNMODIFIED reference
(PYTHONPATH=/root/reference/pkg/src, build container only).
Output: tests/golden/forward_golden.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vitertile.codes import CodeSpec  # noqa: E402
from vitertile import reference as R  # noqa: E402

out = {}
cases = [("k3", 3, (0o7, 0o5)), ("k7", 7, (0o171, 0o133)), ("k7r3", 7, (0o133, 0o171, 0o165)), ("k9", 9, (0o753, 0o561))]
rng = np.random.default_rng(2011)
for name, k, gens in cases:
    spec = CodeSpec(k, gens)
    f, n = 5, 40
    llrs = rng.integers(-128, 128, size=(f, len(gens), n)).astype(np.float64)
    llrs[0, :, :10] = 0  # ties
    init = rng.integers(-50, 50, size=spec.num_states).astype(np.float64)
    for tag, kw in (("plain", {}), ("renorm", {"renormalize": True}), ("init", {"initial_metrics": init}),
                    ("init_renorm_hist", {"initial_metrics": init, "renormalize": True, "keep_history": True})):
        surv, lam, hist = R.forward_batch(llrs, spec, **kw)
        bits = R.traceback_batch(surv, lam, spec)
        key = f"{name}_{tag}"
        out[key + "_llr"] = llrs.astype(np.int8)
        out[key + "_surv"] = surv
        out[key + "_lam"] = lam
        out[key + "_bits"] = bits
        if hist is not None:
            out[key + "_hist"] = hist
        if "initial_metrics" in kw:
            out[key + "_init"] = init
    frame = rng.integers(-128, 128, size=(len(gens), 30)).astype(np.float64)
    out[f"{name}_decref_llr"] = frame.astype(np.int8)
    out[f"{name}_decref_init"] = init
    out[f"{name}_decref_bits"] = R.decode_reference(frame, spec, initial_metrics=init)
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "forward_golden.npz"), **out)
print(len(out), "arrays")
