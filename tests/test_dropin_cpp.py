"""The C++ drop-in header (include/mgraph_b200.hpp) compiles against the
reference-shaped API and runs the reference's own unit-test cases."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1504_04804_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_test")


def _build():
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(ROOT, "include", "mgraph_b200.hpp")),
            os.path.getmtime(os.path.join(LIBDIR, "libmgraph_b200.so"))):
        return
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src,
                    "-L" + LIBDIR, "-lmgraph_b200", "-Wl,-rpath," + LIBDIR, "-o", BIN],
                   check=True)


def test_dropin_header_compiles_and_host_cases_pass():
    _build()
    r = subprocess.run([BIN, "--host-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
