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
