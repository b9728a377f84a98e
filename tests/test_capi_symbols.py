"""The C-ABI library loads and exports every entry point include/*.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import glob
import os
import re

import pytest

from paper_2201_09827_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(gb_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_the_binding_surface():
    assert set(_lib.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libgcrodr_b200.so missing: run __graft_entry__.build()")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    lib2 = _lib.load()
    assert lib2.gb_version().decode().startswith("gcrodr_b200")


def test_no_gpu_means_loud_failure(monkeypatch):
    lib = _lib.load()
    if lib.gb_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.GpuUnavailable):
        _lib.require_gpu()
