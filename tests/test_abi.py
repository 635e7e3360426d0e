"""The C-ABI library loads on a GPU-less host and exports exactly what include/spst.h
declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2212_13459_b200 import _native, errors


def header_functions():
    with open(os.path.join(ROOT, "include", "spst.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spst_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), f"libspst.so does not export {n}"
    assert set(names) == set(_native.SIGNATURES), "ctypes signature table out of sync with include/spst.h"


def test_abi_version_and_status_strings():
    lib = _native.lib()
    assert lib.spst_abi_version() == 1
    assert lib.spst_status_string(0) == b"ok"
    assert b"geometry" in lib.spst_status_string(2)


def test_status_codes_map_to_reference_exceptions():
    for code, exc in [(1, errors.ShapeError), (2, errors.GeometryError), (3, errors.ConfigError),
                      (4, errors.NonFiniteError), (6, MemoryError), (7, NotImplementedError), (8, errors.EmptyError)]:
        with pytest.raises(exc):
            _native.check(code)
    _native.check(0)


def test_built_for_sm100a_only():
    with os.popen(f"cuobjdump --list-elf {os.path.join(ROOT, 'paper_2212_13459_b200', 'libspst.so')} 2>&1") as pipe:
        out = pipe.read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_create_without_device_fails_loudly():
    """No CUDA device here: the product path must raise, never fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    from paper_2212_13459_b200.device import Engine
    from paper_2212_13459_b200.spec import tinynet
    with pytest.raises(RuntimeError):
        Engine(tinynet(0))
