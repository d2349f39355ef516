import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def pytest_sessionstart(session):
    """A fresh checkout has no built library: build it (nvcc cross-compiles sm_100a
    without a GPU) so the C-ABI tests run; a GPU box receives the prebuilt .so."""
    lib = os.path.join(ROOT, "paper_2011_13579_b200", "libvitertile_b200.so")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(lib) and os.path.exists(nvcc):
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def golden():
    z = np.load(GOLDEN)
    index = json.loads(bytes(z["index_json"]).decode())
    return z, index


def golden_cases(kind):
    z = np.load(GOLDEN)
    index = json.loads(bytes(z["index_json"]).decode())
    return [c for c in index["cases"] if c["kind"] == kind], index["codes"]


def code_params(codes, name):
    k, polys = codes[name]
    return int(k), tuple(int(p, 8) for p in polys)


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
