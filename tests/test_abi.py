"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/kerntune_b200.h declares (no compute calls here)."""

import ctypes
import pathlib
import re

import pytest

from paper_2102_04199_b200 import _lib

HEADER = pathlib.Path(__file__).resolve().parent.parent / "include" / "kerntune_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\**\s+\**(kt_[a-z0-9_]+)\s*\(",
                                 text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2102_04199_b200.build import build

    build()
    return _lib.load()


def test_header_and_binding_agree():
    assert declared_functions() == _lib.exported_symbols()


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.kt_version() == 1
    assert lib.kt_last_error() == b""


def test_struct_layouts_match_c(lib):
    # offsets of the last members pin the whole layout (checked against gcc's sizeof)
    assert ctypes.sizeof(_lib.SpecTable) == 47384
    assert _lib.SpecTable.fstd.offset == 47000
    assert _lib.SpecTable.choice_off.offset == 47352
    assert ctypes.sizeof(_lib.Dims) == 128


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}


def test_error_codes_map_to_reference_taxonomy():
    from paper_2102_04199_b200.errors import DomainError, NumericError

    for code in (_lib.KT_E_SHAPE, _lib.KT_E_EMPTY, _lib.KT_E_RANGE, _lib.KT_E_UNSUPPORTED, _lib.KT_E_ARG):
        with pytest.raises(DomainError):
            _lib.check(code, "x")
    for code in (_lib.KT_E_CUDA, _lib.KT_E_NUMERIC):
        with pytest.raises(NumericError):
            _lib.check(code, "x")


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: a missing extension raises instead of degrading."""
    from paper_2102_04199_b200 import _lib
    from paper_2102_04199_b200.errors import NumericError

    with pytest.raises(NumericError):
        _lib.load(tmp_path / "libkerntune_b200.so")
