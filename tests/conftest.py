"""Shared fixtures.  `-m gpu` tests need a B200 (sm_100a) and the in-tree
libsemimat_b200.so; everything else runs on the CPU build container."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")


@pytest.fixture(scope="session")
def small_cases():
    manifest = json.loads((GOLDEN / "small_cases.json").read_text())
    arrays = np.load(GOLDEN / "small_cases.npz")
    out = []
    for meta in manifest:
        prefix = meta["name"] + "__"
        arrs = {k[len(prefix):]: arrays[k] for k in arrays.files if k.startswith(prefix)}
        out.append((meta, arrs))
    return out


@pytest.fixture(scope="session")
def samples():
    return json.loads((GOLDEN / "samples.json").read_text())


@pytest.fixture(scope="session")
def config_digests():
    return json.loads((GOLDEN / "config_digests.json").read_text())


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle
