import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    # always (re)build the library: make's dependency tracking makes this a
    # no-op when it is current, and a stale .so must never be tested against
    # newer sources (nvcc cross-compiles sm_100a without a GPU)
    import subprocess
    subprocess.run(["make", "-C", str(ROOT / "paper_2105_10332_b200" / "csrc"), "-j8"], check=True,
                   capture_output=True)


@pytest.fixture(scope="session")
def oracle():
    from oracle_bind import Restated
    try:
        return Restated()
    except FileNotFoundError:
        import subprocess
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "restated"], check=True, capture_output=True)
        return Restated()


@pytest.fixture(scope="session")
def reference():
    from oracle_bind import reference_or_none
    r = reference_or_none()
    if r is None:
        pytest.skip("reference library oracle/_ref not built here")
    return r


@pytest.fixture(scope="session")
def sg():
    import paper_2105_10332_b200 as sg
    return sg
