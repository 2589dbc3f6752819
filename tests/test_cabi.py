"""CPU checks of the C ABI: the library loads without a GPU and exports exactly
what include/tlg_b200.h declares; error paths that need no device work."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tlg_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tlg_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    from paper_2011_12895_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        pytest.skip("library not built")
    return _capi.lib()


def test_header_declares_the_python_binding_surface():
    from paper_2011_12895_b200 import _capi
    assert sorted(_capi.EXPORTS) == declared_functions()


def test_library_exports_every_declared_symbol(L):
    for name in declared_functions():
        assert hasattr(L, name), name


def test_version_and_no_device_error(L):
    assert b"sm_100a" in L.tlg_version()
    from paper_2011_12895_b200._capi import LearnerConfig, PolicyShape
    cfg = LearnerConfig(0, 1, 0.9, 0.999, 1e-8, 4, 3, 0, 0, 0)
    shape = PolicyShape.make("mlp", 3, 2, (6,))  # hidden width not a multiple of 4
    h = C.c_void_p()
    rc = L.tlg_learner_create(C.byref(cfg), C.byref(shape), C.byref(h))
    assert rc == 1  # TLG_INVALID_ARGUMENT raised before any device work
    assert b"multiples of 4" in L.tlg_last_error()
