"""The C-ABI library loads and exports every symbol declared in include/coverblip_b200.h
(no compute calls: runs on CPU)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "coverblip_b200.h")
LIB = os.path.join(ROOT, "paper_1810_01967_b200", "libcoverblip_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cbb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1810_01967_b200", "csrc")],
                       check=True)
    return LIB


def test_header_declares_api():
    names = declared()
    for must in ("cbb_project_cone_exact", "cbb_project_step", "cbb_dict_prepare",
                 "cbb_op_apply", "cbb_op_adjoint", "cbb_argmax_select"):
        assert must in names


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (cbb_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(built):
    from paper_1810_01967_b200 import _lib
    lib = _lib.load()
    assert set(_lib.SIGNATURES) == set(declared())
    assert lib.cbb_abi_version() == 3
    # sizes are pure host arithmetic
    assert lib.cbb_project_workspace_bytes(1 << 20, 10) > (1 << 20) * 64
    assert lib.cbb_dict_storage_bytes(1 << 17, 10) >= (1 << 17) * 10 * 16


def test_sass_has_tcgen05_and_bulk_copy(built):
    sass = subprocess.run(["cuobjdump", "-sass", built], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass, "tcgen05.mma missing from the matched-filter kernel"
    assert "LDTM" in sass and "UBLKCP" in sass
