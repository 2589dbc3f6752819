import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "lib", "libtlg_oracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "lib"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    from oracle_ffi import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_ffi import try_ref
    r = try_ref()
    if r is None:
        pytest.skip("oracle/_ref not built (reference sources unavailable here)")
    return r


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")

    def load(name):
        return np.load(os.path.join(d, name + ".npz"))
    return load


@pytest.fixture(scope="session")
def tlg():
    """The product library (CUDA path).  GPU tests only."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2011_12895_b200 as p
    return p
