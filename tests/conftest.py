import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from helpers import load_gz  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librlx.so")


@pytest.fixture(scope="session")
def golden_schedules():
    return load_gz("schedules.json.gz")


@pytest.fixture(scope="session")
def golden_keys():
    return load_gz("keys.json.gz")


@pytest.fixture(scope="session")
def golden_schedules_knobs():
    return load_gz("schedules_knobs.json.gz")


@pytest.fixture(scope="session")
def Evaluator():
    """The device chooser class (librlx.so through the C-ABI)."""
    from paper_2604_23838_b200.native import Evaluator as E

    return E
