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


def test_host_side_entry_points_validate_arguments(lib):
    """kt_sa_draws is host-side (no GPU): its argument checks return the documented codes."""
    import ctypes

    import numpy as np

    pcg = np.array([0, 12345, 0, 6789], dtype=np.uint64)  # (odd increment: a valid PCG64 state)
    has = np.zeros(1, dtype=np.int32)
    ui = np.zeros(1, dtype=np.uint32)
    out = [np.zeros((2, 3), dtype=dt) for dt in (np.int32, np.uint8, np.int32, np.int32, np.float64)]
    p = lambda a: a.ctypes.data  # noqa: E731
    cards = np.array([3, 0], dtype=np.int32)
    assert lib.kt_sa_draws(None, p(has), p(ui), 2, 3, 2, p(cards), *map(p, out)) == 7  # KT_E_ARG
    assert lib.kt_sa_draws(p(pcg), p(has), p(ui), 2, 3, 0, p(cards), *map(p, out)) == 1  # KT_E_SHAPE
    assert lib.kt_sa_draws(p(pcg), p(has), p(ui), 2, 3, 2, p(cards), *map(p, out)) == 3  # KT_E_RANGE (empty knob)
    assert b"empty knob" in ctypes.string_at(lib.kt_last_error())
    cards[1] = 4
    even = np.array([0, 12345, 0, 6788], dtype=np.uint64)
    assert lib.kt_sa_draws(p(even), p(has), p(ui), 2, 3, 2, p(cards), *map(p, out)) == 7  # even increment
    assert lib.kt_sa_draws(p(pcg), p(has), p(ui), 2, 3, 2, p(cards), *map(p, out)) == 0
