import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity through the C-ABI")
    # The CPU checkers are test infrastructure; build them if this checkout has
    # not (gcc is present here and on the GPU box).  oracle/_ref needs the
    # reference tree, so it is only (re)built where that exists.
    port = os.path.join(ROOT, "oracle", "_build", "libsk_oracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "libsemikern_ref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port.get()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref/libsemikern_ref.so not built (reference tree absent)")
    return Ref.get()


@pytest.fixture(scope="session")
def sk():
    """The product package; GPU tests only."""
    import paper_1708_02937_b200 as sk
    sk.default_context()  # raises CudaError without a device -- no fallback
    return sk
