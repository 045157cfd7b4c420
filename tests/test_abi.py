"""CPU-side checks of the C-ABI boundary: the shared library is built for
sm_100a, loads without a GPU, and exports every entry point declared in
include/adrom_b200.h."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "adrom_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(adrom_[a-z0-9_]+)\s*\(", text))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2605_28684_b200 import _build
    return _build.build()


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert {"adrom_rhs", "adrom_implicit_step", "adrom_isvd_update", "adrom_project"} <= syms


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(adrom_[a-z0-9_]+)\b", out))
    missing = declared_symbols() - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"


def test_ctypes_signatures_cover_header(lib_path):
    from paper_2605_28684_b200 import _lib
    assert declared_symbols() <= set(_lib.SIGNATURES), \
        sorted(declared_symbols() - set(_lib.SIGNATURES))
    assert _lib.exported_symbols(lib_path) == set(_lib.SIGNATURES)


def test_library_loads_and_reports_abi_version(lib_path):
    import ctypes
    lib = ctypes.CDLL(str(lib_path))
    assert lib.adrom_abi_version() == 2


def test_kernels_are_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib_path)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
