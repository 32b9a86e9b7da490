import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


try:  # same profile as the reference suite (tests/conftest.py:5-11)
    from hypothesis import HealthCheck, settings

    settings.register_profile("default", max_examples=25, deadline=None,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("default")
except ImportError:  # pragma: no cover
    pass


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


@pytest.fixture(scope="session")
def knn_golden():
    g = np.load(GOLDEN / "knn_cases.npz")
    import json
    cases = []
    for ci in range(int(g["ncases"])):
        p = f"c{ci}/"
        cases.append(dict(spec=json.loads(str(g[p + "spec"])), refs=g[p + "refs"], queries=g[p + "queries"],
                          keys=g[p + "keys"], counts=g[p + "counts"], visited=g[p + "visited"],
                          seq_len=g[p + "seq_len"], seq=g[p + "seq"], digest=str(g[p + "digest"])))
    return cases


@pytest.fixture(scope="session")
def gpu_device():
    from paper_1512_02831_b200 import DeviceSpec, GpuDevice
    dev = GpuDevice(DeviceSpec(cuda_device=0))
    yield dev
    dev.close()
