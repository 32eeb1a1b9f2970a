"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest run on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (sm_100a)")


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_trace_meshes():
    from paper_2504_21719_b200.geometry import Mesh
    g = golden("trace.npz")
    return [Mesh(g[f"verts_{i}"], g[f"tris_{i}"], object_id=int(g[f"oid_{i}"]))
            for i in range(int(g["nmesh"]))]


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
