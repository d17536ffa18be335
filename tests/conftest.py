import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size configuration runs")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


@pytest.fixture(scope="session")
def oracle_c():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import REF_SO, Reference
    if not REF_SO.exists():
        pytest.skip("compiled reference (oracle/_ref) not built here")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    from paper_1706_06664_b200 import _native as N
    if not N.dev().ace_device_available():
        pytest.fail("GPU test run without a usable CUDA device")
    import torch
    return torch
