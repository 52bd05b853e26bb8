import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # The C restatement (checker) is a few hundred lines of C: build it if
    # this checkout does not carry the prebuilt .so yet.
    so = os.path.join(ROOT, "oracle", "_build", "libtt_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def ctx():
    from paper_2402_02361_b200.tiletune import Context
    c = Context(0)
    yield c
    c.close()
