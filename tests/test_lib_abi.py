"""The C-ABI library loads and exports every symbol include/*.h declares.
CPU only: no compute calls."""

import ctypes
import os
import re

from paper_2302_05164_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "scantherm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_typed():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 25
    typed = {n for n, _, _ in _lib.SIGNATURES}
    for n in names:
        assert hasattr(lib, n), n
        assert n in typed, f"{n} has no ctypes signature"


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.StBeam) == 40
    assert ctypes.sizeof(_lib.StMaterial) == 10 * 8
    assert ctypes.sizeof(_lib.StBoundary) == 11 * 8
    assert ctypes.sizeof(_lib.StParams) == (10 + 11 + 3) * 8
    from paper_2302_05164_b200.physics import BEAM_DTYPE
    assert BEAM_DTYPE.itemsize == 40


def test_version_and_error_plumbing_without_gpu():
    lib = _lib.load()
    assert lib.st_version() >= 100
    n = ctypes.c_int()
    rc = lib.st_device_count(ctypes.byref(n))
    if rc != 0:
        assert lib.st_last_error()  # message explains the failure
