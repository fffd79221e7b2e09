"""Shared fixtures. ``@pytest.mark.gpu`` marks tests that need a B200."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_npz(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def codec_golden():
    return load_json("codec_cases.json"), load_npz("codec_cases.npz")


@pytest.fixture(scope="session")
def stream_golden():
    return load_json("streams.json"), load_npz("streams.npz")


@pytest.fixture(scope="session")
def traces():
    return load_json("train_traces.json")
