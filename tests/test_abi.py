"""CPU tests of the C-ABI boundary: the library loads without a GPU and
exports exactly the entry points include/mcs_abi.h declares, with the
argument counts the ctypes binding uses; layout queries agree with the
Python packers."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2207_08481_b200 import _abi, engine
from paper_2207_08481_b200.refblocks import local_sizes

HEADER = os.path.join(ROOT, "include", "mcs_abi.h")


def header_decls():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    out = {}
    for m in re.finditer(r"\bint\s+(mcs_\w+)\s*\(([^)]*)\)\s*;", txt):
        args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    decls = header_decls()
    assert len(decls) >= 20
    for name in decls:
        assert hasattr(lib, name), name


def test_binding_matches_header():
    decls = header_decls()
    assert set(decls) == set(_abi.SIGNATURES)
    for name, nargs in decls.items():
        assert len(_abi.SIGNATURES[name]) == nargs, name


@pytest.mark.parametrize("k", [2, 3, 4, 5, 6])
def test_layout_queries(k):
    lib = ctypes.CDLL(_abi.LIB_PATH)
    assert lib.mcs_record_len(k) == engine.record_layout(k)["len"]
    assert lib.mcs_srec_len(k) == engine.srecord_layout(k)["len"]
    assert lib.mcs_st_stride(k) == engine.st_stride(k)
    z = local_sizes(k)
    ni, nc = z["n_int"], z["ncpl"]
    assert lib.mcs_ext_stride(k) == engine.packed_stride(0) + \
        ((ni * nc + ni * (ni + 1) // 2 + 1) & ~1)
    assert lib.mcs_sd_stride(k) == engine.packed_stride(nc)


def test_product_path_has_no_cpu_fallback(monkeypatch, tmp_path):
    """With the library missing the product raises instead of computing."""
    monkeypatch.setattr(_abi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(_abi.McsError):
        _abi.lib()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2207_08481_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "from oracle" not in src and "import oracle" not in src, fn
