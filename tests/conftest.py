import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under `-m gpu` on the GPU box)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference library itself (oracle/_ref/libref.so); skipped if not built."""
    from oracle.bindings import Reference
    path = os.path.join(ROOT, "oracle", "_ref", "libref.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/libref.so not built (needs /root/reference at build time)")
    return Reference(path)


@pytest.fixture(scope="session")
def golden():
    out = {}
    for name in ("models", "evolve", "sweep", "kat"):
        with np.load(os.path.join(GOLDEN, f"golden_{name}.npz")) as z:
            out[name] = {k: z[k] for k in z.files}
    return out


@pytest.fixture(scope="session")
def lbg():
    import paper_2603_18052_b200 as lbg
    lbg.lib()
    return lbg
