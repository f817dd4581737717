"""The C-ABI library builds, loads and exports every symbol the header declares."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1912_07962_b200 import _lib, build
    build.build()
    return _lib.lib()


def test_header_symbols_exported(lib):
    from paper_1912_07962_b200 import _lib
    with open(os.path.join(ROOT, "include", "slimb200.h")) as fh:
        text = fh.read()
    declared = set(re.findall(r"\b(slim_[a-z0-9_]+)\s*\(", text))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version(lib):
    assert lib.slim_abi_version() == 1


def test_create_validation_without_gpu(lib):
    """Argument validation runs before any device call (ValueError mapping)."""
    import ctypes as C
    from paper_1912_07962_b200 import _lib
    d = _lib.SlimDesc()
    d.n_rows, d.n_cols, d.block_rows, d.memory_r = 10, 4, 3, 0
    ctx = C.c_void_p()
    rc = lib.slim_create(C.byref(ctx), C.byref(d))
    assert rc == _lib.SLIM_EINVAL
    with pytest.raises(ValueError, match="not divisible"):
        _lib.check(rc, None)


def test_product_does_not_import_oracle():
    """The product never imports, includes or loads anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1912_07962_b200")
    imp = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b)|importlib.*oracle|"
                     r"sys\.path.*oracle", re.M)
    inc = re.compile(r'#include\s+[<"][^>"]*oracle')
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                assert not imp.search(open(path).read()), path
            elif f.endswith((".cu", ".cpp", ".h", ".cuh")):
                assert not inc.search(open(path).read()), path
