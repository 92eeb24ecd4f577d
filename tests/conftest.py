import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference built in place)")


def _has_ref():
    from oracle import ref
    return ref.available()


@pytest.fixture(scope="session")
def refmod():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref/libcdg_ref.so not built (reference sources absent)")
    return ref


@pytest.fixture(scope="session")
def gpu_lib():
    """The product library; GPU tests fail (not skip) when it is missing."""
    from paper_1208_4772_b200 import gpu
    gpu.lib()
    return gpu
