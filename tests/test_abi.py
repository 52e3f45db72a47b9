"""The C-ABI library loads and exports every function include/lofp.h declares; host-side
argument validation that happens before any device work (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "lofp.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lofp_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_26408_b200 import _build
    _build.build()
    return ctypes.CDLL(_build.LIB)


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert {"lofp_create", "lofp_amplitudes", "lofp_destroy", "lofp_status_string", "lofp_last_error"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    from paper_2510_26408_b200 import EXPORTS
    assert sorted(EXPORTS) == names


def test_status_strings(lib):
    lib.lofp_status_string.restype = ctypes.c_char_p
    assert lib.lofp_status_string(0) == b"ok"
    assert lib.lofp_status_string(2) == b"unsupported"


def test_create_validation_without_device():
    from paper_2510_26408_b200 import Circuit, LofpError
    bad = [
        (4, [[(0, 1, 0.1, 0.2), (1, 2, 0.3, 0.4)]], 1),      # overlapping pairs
        (4, [[(0, 4, 0.1, 0.2)]], 1),                        # mode out of range
        (4, [[(1, 1, 0.1, 0.2)]], 1),                        # a == b
        (4, [[(0, 1, float("inf"), 0.2)]], 1),               # non-finite angle
        (0, [], 1),                                          # no modes
        (129, [], 2),                                        # too many modes
    ]
    for M, layers, want in bad:
        with pytest.raises(LofpError) as e:
            Circuit(M, layers)
        assert e.value.status == want, (M, layers)


def test_null_arguments(lib):
    lib.lofp_create.restype = ctypes.c_int
    assert lib.lofp_create(4, 0, None, None, None) == 1
    h = ctypes.c_void_p()
    assert lib.lofp_create(4, 1, None, None, ctypes.byref(h)) == 1
    lib.lofp_destroy(None)
    lib.lofp_amplitudes.restype = ctypes.c_int
    assert lib.lofp_amplitudes(None, None, 0, None, None, None) == 1
