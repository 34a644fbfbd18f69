"""Shared fixtures.  `-m gpu` tests need a CUDA device and libqsv.so; every
other test runs on CPU (oracle vs golden vectors, parser, scheduler emulation,
C-ABI load checks, multi-process host logic over gloo)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).parent))

GOLDEN = Path(__file__).parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libqsv.so")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "programs.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "states.npz") as f:
        return {k: f[k] for k in f.files}


def program_text(golden, name):
    if name in golden["programs"]:
        return golden["programs"][name]["text"]
    if name in golden["random_programs"]:
        return golden["random_programs"][name]["text"]
    import re

    from paper_2008_07140_b200.rqc import RqcConfig, generate_rqc

    m = re.match(r"rqc_(\d+)x(\d+)_(\d+)_(\d+)", name)
    return generate_rqc(RqcConfig(*map(int, m.groups())))
