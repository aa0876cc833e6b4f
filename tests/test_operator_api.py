"""The operator API (include/mgraph_b200_spec.cuh): user-defined primitives —
PrimitiveSpec<State, Dev> + run_primitive, the reference's engine.hpp:587-626,
712 — compiled with nvcc against the engine templates and linked to
libmgraph_b200.so.  tests/cpp/spec_test.cu ports the reference's custom-spec
callers: the worker-failure case (test_engine.cpp:272-287) and the
per-superstep latency microbench (cost_model.cpp:76-112), plus a spec shipping
8 + 8 associates per record and a broadcast-mode spec."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1504_04804_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "spec_test.cu")
BIN = os.path.join(ROOT, "tests", "cpp", "spec_test")


def build():
    deps = [SRC, os.path.join(ROOT, "include", "mgraph_b200_spec.cuh"),
            os.path.join(ROOT, "include", "mgraph_b200.hpp"),
            os.path.join(LIBDIR, "libmgraph_b200.so")]
    csrc = os.path.join(LIBDIR, "csrc")
    deps += [os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cuh", ".hpp"))]
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(os.path.getmtime(d) for d in deps):
        return
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-O2", "-lineinfo",
                    "-gencode", "arch=compute_100a,code=sm_100a", "--expt-relaxed-constexpr",
                    "-I" + os.path.join(ROOT, "include"), "-I" + csrc, SRC, "-L" + LIBDIR,
                    "-lmgraph_b200", "-Xlinker", "-rpath=" + LIBDIR, "-o", BIN], check=True,
                   capture_output=True)


def test_user_spec_compiles_against_the_engine_header():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_user_specs_run_on_gpu():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
    lat = [float(x) for x in re.findall(r"per_iter_us=([\d.]+)", r.stdout)]
    assert len(lat) == 3 and all(0 < x < 5000 for x in lat)
