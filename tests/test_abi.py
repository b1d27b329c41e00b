"""The C ABI library loads and exports every symbol include/jt_b200.h declares
(no compute calls: this runs on the CPU-only CI host)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "jt_b200.h")
LIB = os.path.join(ROOT, "paper_1202_3777_b200", "libjtb200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(jt_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_1202_3777_b200", "csrc")])
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_table_covers_header():
    from paper_1202_3777_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == declared_functions()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string(lib):
    lib.jt_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.jt_version()


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_1202_3777_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
