"""Shared test setup: the `gpu` marker and golden-fixture loaders."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_perm():
    with open(os.path.join(GOLDEN, "golden_perm.json")) as fh:
        return json.load(fh)


def rel_l2(got, want) -> float:
    import numpy as np
    got = np.asarray(got, dtype=np.complex128)
    want = np.asarray(want, dtype=np.complex128)
    den = float(np.linalg.norm(want))
    num = float(np.linalg.norm(got - want))
    return num / den if den > 0 else num


def golden_amps(case):
    import numpy as np
    return np.array([complex(re, im) for re, im in case["amps"]])


@pytest.fixture(scope="session")
def golden_sampler():
    with open(os.path.join(GOLDEN, "golden_sampler.json")) as fh:
        return json.load(fh)
