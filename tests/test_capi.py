"""CPU checks of the C ABI library: it loads without a GPU and exports every
symbol include/walkjoin_b200.h declares; the ctypes table matches the header."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "walkjoin_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int)\s*(wj_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2202_13538_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_path():
    names = _declared()
    for must in ("wj_sample_walks", "wj_rpe_count", "wj_rpe_fill", "wj_intern_insert",
                 "wj_intern_assign", "wj_join", "wj_gather_rpe", "wj_export_dicts", "wj_lookup",
                 "wj_last_error", "wj_abi_version"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_abi_version_and_error_string(lib):
    lib.wj_abi_version.restype = ctypes.c_int
    assert lib.wj_abi_version() == 1
    lib.wj_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.wj_last_error(), bytes)


def test_argument_errors_without_gpu(lib):
    """Argument validation happens before any launch, so it works on CPU."""
    from paper_2202_13538_b200 import _lib

    _lib.load()
    with pytest.raises(ValueError, match="num_walks"):
        _lib.call("wj_sample_walks", None, 4, None, 10, 0, 10, 0, 3, 1, None, None, None)
    with pytest.raises(ValueError, match="idxptr_bytes"):
        _lib.call("wj_sample_walks", None, 2, None, 10, 0, 10, 5, 3, 1, None, None, None)
    with pytest.raises(ValueError, match="range"):
        _lib.call("wj_sample_walks", None, 4, None, 10, 5, 11, 5, 3, 1, None, None, None)
    with pytest.raises(NotImplementedError, match="4096"):
        _lib.call("wj_rpe_count", None, 0, 2000, 4, 10, None, None)
    with pytest.raises(ValueError, match="power of two"):
        _lib.call("wj_intern_insert", None, None, None, 1, 0, None, None, 3, None, None)
    with pytest.raises(NotImplementedError, match="arity"):
        _lib.call("wj_join", None, 1, 5, None, None, None, None, None, 2, 2, 1, None, 1, None,
                  None, None, 0, 10, None)


def test_ctypes_table_matches_header():
    from paper_2202_13538_b200 import _lib

    src = open(HEADER).read()
    for name, argtypes in _lib.SIGNATURES.items():
        m = re.search(r"\b" + name + r"\s*\(([^)]*)\)", src, re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(argtypes), name
