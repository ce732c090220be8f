import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def mask_blobs():
    return dict(np.load(os.path.join(GOLDEN, "mask_blobs.npz")))


@pytest.fixture(scope="session")
def philox_vectors():
    return dict(np.load(os.path.join(GOLDEN, "philox_vectors.npz")))


@pytest.fixture(scope="session")
def attn_arrays():
    return dict(np.load(os.path.join(GOLDEN, "attention_arrays.npz")))


@pytest.fixture(scope="session")
def rgo():
    import paper_2410_07531_b200 as r
    return r


@pytest.fixture(scope="session")
def cuda(rgo):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test needs a CUDA device")
    return torch.device("cuda")
