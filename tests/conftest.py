"""Shared fixtures. ``-m gpu`` tests need a B200; everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref); built here when the
    reference sources are mounted, skipped on hosts that have neither."""
    from oracle import pyoracle
    if not pyoracle.ref_available() and os.path.isdir(os.path.join(pyoracle.REF_SRC, "src")):
        pyoracle.build(ref=True)
    if not pyoracle.ref_available():
        pytest.skip("reference library (oracle/_ref) not built on this host")
    return pyoracle.RefLib()


@pytest.fixture(scope="session")
def coracle():
    from oracle import pyoracle
    pyoracle.build(ref=False)
    return pyoracle.COracle()


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2511_20432_b200 as tg
    return tg.Context(0)


@pytest.fixture(scope="session")
def configs():
    from paper_2511_20432_b200 import workloads
    return workloads.write_configs(os.path.join(ROOT, "configs"))
