import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100) device")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_scene_arrays(g):
    """oracle.SceneArrays from a golden npz (host softplus like render.py:52)."""
    from oracle import oracle as orc
    from paper_2502_01157_b200.scene import softplus

    return orc.SceneArrays(g["positions"], g["offsets"].astype(np.int64),
                           g["neighbors"].astype(np.int64), softplus(g["raw_density"]), g["sh"],
                           g["background"])


def golden_scene(g):
    from paper_2502_01157_b200.scene import AdjacencyGraph, FoamScene

    adj = AdjacencyGraph(g["positions"], g["offsets"].astype(np.int64),
                         g["neighbors"].astype(np.int64))
    return FoamScene(g["positions"], g["raw_density"], g["sh"].reshape(-1, 16, 3),
                     g["background"], adj)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_01157_b200 import _lib

    lib = _lib.load()
    assert lib.rfb_device_ok() == 1, "current device is not sm_100"
    return True
