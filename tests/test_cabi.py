"""The C-ABI library builds, loads and exports every entry point include/dk_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "dk_b200.h")
LIB = os.path.join(REPO, "paper_2406_18109_b200", "libdk_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dk_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_18109_b200.build import build

    build()
    stub = "/usr/local/cuda/lib64/stubs/libcuda.so"
    try:
        ctypes.CDLL("libcuda.so.1", mode=ctypes.RTLD_GLOBAL)
    except OSError:
        ctypes.CDLL(stub, mode=ctypes.RTLD_GLOBAL)  # CPU box: resolve libcuda.so.1 to the stub
    return ctypes.CDLL(LIB)


def test_header_declares_the_abi():
    names = declared()
    assert "dk_launch" in names and "dk_kernel_compile" in names and "dk_comm_exchange" in names
    assert len(names) >= 35


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2406_18109_b200.runtime import EXPORTED

    assert sorted(EXPORTED) == declared()


def test_sm100a_code_in_library(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_without_a_device(lib):
    lib.dk_last_error.restype = ctypes.c_char_p
    rc = lib.dk_store_free(ctypes.c_int64(1))
    assert rc == 5  # DK_ERR_STATE: not initialised
    assert b"dk_init" in lib.dk_last_error()
