import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # native artefacts are git-ignored: (re)build them in-tree if missing or stale
    import build_native
    build_native.build_synth()
    build_native.build_oracle()
    if os.environ.get("MS_SKIP_LIBMS_BUILD") != "1":
        build_native.build_libms()


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def as_int(x):
    return int(x, 16) if isinstance(x, str) else int(x)


@pytest.fixture(scope="session")
def worked():
    return load_golden("worked_examples.json")


@pytest.fixture(scope="session")
def paper_pins():
    return load_golden("paper_pins.json")


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
