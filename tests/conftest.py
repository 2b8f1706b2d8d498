import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_errors():
    return json.loads((GOLDEN / "golden_errors.json").read_text())


@pytest.fixture(scope="session")
def golden_groups():
    return json.loads((GOLDEN / "golden_groups.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2506_19656_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


@pytest.fixture
def variant_sel():
    """Select kernel variants (cv_set_variant) for one test; restores the defaults."""
    from paper_2506_19656_b200 import _lib

    defaults = {"gram_tiles": 0, "gram_nt": 64, "proj_nopf": 0, "proj12": 1, "gram_checks": 0, "gram12": 1, "qp_px1": 0, "qp_runtime_c": 0,
                "eval_kernel": 0}

    def sel(variants: dict):
        for k, v in variants.items():
            _lib.set_variant(k, v)

    yield sel
    for k, v in defaults.items():
        _lib.set_variant(k, v)
