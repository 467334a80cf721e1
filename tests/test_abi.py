"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/dwconv.h declares, and validates descriptors before touching a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1803_09926_b200 import build, _lib
    build.build()
    return _lib.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "dwconv.h")).read()
    return sorted(set(re.findall(r"DWCONV_API\s+[\w\s\*]+?\b(dwconv_\w+)\s*\(", src)))


def test_header_declares_the_three_passes():
    names = _declared()
    for n in ("dwconv_fwd", "dwconv_bwd_data", "dwconv_bwd_filter", "dwconv_bwd_filter_workspace_bytes"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    from paper_1803_09926_b200 import _lib
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.FUNCTIONS)
    assert lib.dwconv_abi_version() == 2


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1803_09926_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "dw_oracle" not in txt, f


def _desc(**kw):
    from paper_1803_09926_b200.ops import make_desc
    a = dict(n=2, c=8, h=16, w=16, multiplier=1, kernel=3, stride=1, padding=1, layout=0, dtype=0)
    a.update(kw)
    return make_desc(a["n"], a["c"], a["h"], a["w"], a["multiplier"], a["kernel"], a["stride"], a["padding"],
                     a["layout"], a["dtype"])


def test_output_shape(lib):
    from paper_1803_09926_b200.ops import output_shape
    assert output_shape(_desc()) == (16, 16)
    assert output_shape(_desc(h=112, w=112, stride=2)) == (56, 56)
    assert output_shape(_desc(h=7, w=9, kernel=(3, 5), stride=(1, 2), padding=(1, 0))) == (7, 3)


@pytest.mark.parametrize("bad,status", [
    (dict(n=-1), 2), (dict(c=0), 2), (dict(h=0), 2), (dict(multiplier=0), 2), (dict(kernel=0), 2),
    (dict(stride=0), 2), (dict(padding=-1), 2), (dict(layout=7), 2), (dict(dtype=3), 2),
    (dict(h=2, w=2, kernel=5, padding=0), 3),
])
def test_validation_errors(lib, bad, status):
    d = _desc(**bad)
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    assert lib.dwconv_output_shape(ctypes.byref(d), ctypes.byref(ho), ctypes.byref(wo)) == status
    # the compute entry points validate before any device work (no GPU here)
    assert lib.dwconv_fwd(ctypes.byref(d), None, None, None, None) == status


def test_null_and_misaligned_pointers(lib):
    d = _desc()
    assert lib.dwconv_fwd(ctypes.byref(d), None, None, None, None) == 1
    assert lib.dwconv_fwd(ctypes.byref(d), ctypes.c_void_p(4098), ctypes.c_void_p(4096),
                          ctypes.c_void_p(4096), None) == 4
    # N == 0 is valid and enqueues nothing (no device needed)
    d0 = _desc(n=0)
    assert lib.dwconv_fwd(ctypes.byref(d0), None, ctypes.c_void_p(4096), None, None) == 0
    assert lib.dwconv_bwd_data(ctypes.byref(d0), None, ctypes.c_void_p(4096), None, None) == 0


def test_status_strings(lib):
    from paper_1803_09926_b200._lib import status_string
    assert status_string(3) == "kernel exceeds padded input"
    assert status_string(0) == "ok"
    assert status_string(99) == "unknown status"
