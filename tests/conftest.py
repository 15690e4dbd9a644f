import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def built_lib():
    from paper_2501_11592_b200 import build

    return build.build()


@pytest.fixture(scope="session")
def gpu_available(built_lib):
    import paper_2501_11592_b200 as cl

    n = cl.lib().cl_device_count()
    if n == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return n
