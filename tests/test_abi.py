"""CPU-side checks of the C-ABI boundary: the library loads and exports every
entry point include/vfpi.h declares; struct layouts agree with the header.
No compute calls (there is no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vfpi.h")
LIB = os.path.join(ROOT, "paper_2201_09212_b200", "libvfpi.so")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vfpi_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2201_09212_b200.build import build

        build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    names = declared()
    for must in ("vfpi_create", "vfpi_solve", "vfpi_solve_device", "vfpi_wait", "vfpi_spmv", "vfpi_apply_jc",
                 "vfpi_apply_jc_t", "vfpi_contact_solve_oneshot", "vfpi_step_matrix_frobenius"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_sizes_match_ctypes_mirror():
    from paper_2201_09212_b200._lib import VfpiConfig, VfpiResult, VfpiSystem

    assert ctypes.sizeof(VfpiSystem) == 3 * 8 + 10 * 8
    assert ctypes.sizeof(VfpiConfig) == 6 * 4 + 5 * 8
    assert ctypes.sizeof(VfpiResult) == 5 * 8 + 4 * 4 + 3 * 8


def test_version_and_no_device_behaviour(lib):
    lib.vfpi_version.restype = ctypes.c_int
    assert lib.vfpi_version() == 1
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by -m gpu tests")
    h = ctypes.c_void_p()
    lib.vfpi_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.vfpi_create(0, ctypes.byref(h)) == 5  # VFPI_CUDA_ERROR: no CPU fallback
    assert not h.value


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2201_09212_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def _decls_outside_comments():
    txt = re.sub(r"/\*.*?\*/", " ", open(HEADER).read(), flags=re.S)
    txt = re.sub(r"//[^\n]*", " ", txt)
    return sorted(set(re.findall(r"\b(vfpi_[a-z_0-9]+)\s*\(", txt)))


def test_header_declarations_are_live_code():
    # a declaration swallowed by an unterminated comment would vanish here
    assert _decls_outside_comments() == declared()


@pytest.mark.parametrize("lang", ["c", "c++"])
def test_header_compiles_standalone(lang, tmp_path):
    import shutil
    import subprocess

    cc = shutil.which("gcc" if lang == "c" else "g++")
    if cc is None:
        pytest.skip("no host compiler")
    src = tmp_path / ("t.c" if lang == "c" else "t.cpp")
    src.write_text('#include "vfpi.h"\nint main(void) { return vfpi_version() == 1 ? 0 : 1; }\n')
    r = subprocess.run([cc, "-fsyntax-only", "-Wall", "-Werror", "-I", os.path.dirname(HEADER), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
