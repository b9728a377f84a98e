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


def test_options_block_matches_header():
    """Every gb_options field in include/gcrodr_b200.h is in the ctypes mirror,
    in the same order (the struct crosses the C-ABI by pointer)."""
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "gcrodr_b200.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} gb_options;", hdr, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = [n.strip() for decl in body.split(";") if decl.strip()
             for n in decl.strip().split(None, 1)[1].split(",")]
    assert names == [f[0] for f in _lib.Options._fields_]


@pytest.mark.parametrize("method,restart,cycle,want", [
    ("gmres-ir", "recurrence", "explicit", 0), ("gmres-ir", "explicit", "recurrence", 1),
    ("rgmres-ir", "explicit", "recurrence", 0), ("rgmres-ir", "recurrence", "explicit", 1),
    ("rsgmres-ir", "recurrence", "explicit", 1)])
def test_residual_mode_option(method, restart, cycle, want):
    """Plain GMRES reads restart_residual, GCRO-DR cycle_residual (refine.py:338, 352);
    any value but "recurrence" means the explicit s - A~ x (gmres.py:292-295)."""
    from paper_2201_09827_b200.precision import PrecisionTriple
    from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

    cfg = RefineConfig(PrecisionTriple.parse("half", "single", "double"), Method.parse(method), m=8,
                       k=3 if "r" == method[0] else 0, restart_residual=restart, cycle_residual=cycle)
    assert make_options(cfg, 100).explicit_residual == want


def test_half_flush_to_zero_refused_loudly():
    """set_half_flush_subnormals (precision.py:118-127) is mirrored; the device
    kernels keep fp16 subnormals, so half solves refuse to run while it is on."""
    import paper_2201_09827_b200 as gb
    from paper_2201_09827_b200.refine import make_options

    cfg = gb.RefineConfig(gb.PrecisionTriple.parse("half", "single", "double"), gb.Method.RGMRES_IR, m=8, k=3)
    assert gb.set_half_flush_subnormals(True) is False
    try:
        assert gb.half_flushes_subnormals()
        with pytest.raises(NotImplementedError):
            make_options(cfg, 100)
        cfg2 = gb.RefineConfig(gb.PrecisionTriple.parse("single", "double", "double"), gb.Method.RGMRES_IR, m=8, k=3)
        make_options(cfg2, 100)
    finally:
        assert gb.set_half_flush_subnormals(False) is True
    make_options(cfg, 100)
