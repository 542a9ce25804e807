"""The header-only C++ shim (include/semikern_b200/semikern.hpp) re-exposes the
reference's namespace semikern over the C-ABI.  CPU: it compiles against the
library.  GPU: the restated reference test cases pass through it."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_1708_02937_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_shim")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           SRC, "-L" + LIBDIR, "-lsk_b200", "-Wl,-rpath," + LIBDIR, "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_shim_compiles_against_the_c_abi(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_reference_cases_pass_through_the_shim(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 of 14 cases failed" in r.stdout
