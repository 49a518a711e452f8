import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: full-size CPU oracle checks (minutes)")


def pytest_collection_modifyitems(config, items):
    import torch

    have_gpu = torch.cuda.is_available()
    for item in items:
        if "gpu" in item.keywords and not have_gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device in this container"))


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "golden_small.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_index():
    import json

    return json.loads((GOLDEN / "golden_small_index.json").read_text())


@pytest.fixture(scope="session")
def digests():
    import json

    return json.loads((GOLDEN / "digests.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O
