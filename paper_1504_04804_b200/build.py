"""Build libmgraph_b200.so in-tree: nvcc for sm_100a (-lineinfo), g++ for the host C++.

    python -m paper_1504_04804_b200.build        # incremental
    python -m paper_1504_04804_b200.build -f     # force

Objects go to paper_1504_04804_b200/build/, the shared object next to this
file so it travels to the GPU box with the repo snapshot.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# MG_BUILD_VARIANT=<name> MG_NVCC_DEFS="-DX=1 ..." builds an experiment variant
# into build_<name>/ and libmgraph_b200_<name>.so (loaded with MG_LIB_PATH)
_VARIANT = os.environ.get("MG_BUILD_VARIANT", "")
OUT_DIR = os.path.join(HERE, "build" + ("_" + _VARIANT if _VARIANT else ""))
LIB = os.path.join(HERE, "libmgraph_b200" + ("_" + _VARIANT if _VARIANT else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas=-v",
                  "--expt-relaxed-constexpr", "-I" + CSRC, "-I" + os.path.join(ROOT, "include")] + \
    os.environ.get("MG_NVCC_DEFS", "").split()
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", "-I" + CSRC,
            "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]

CU = ["plan.cu", "prims.cu", "api.cu", "gen.cu", "fabric.cu"]
CPP = ["host_graph.cpp", "shm_fabric.cpp"]


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))] + \
        [os.path.join(ROOT, "include", "mgraph_b200.h")]


def _stale(obj, src, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def build(force=False, verbose=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    deps = _headers()
    jobs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(OUT_DIR, f + ".o")
        if force or _stale(obj, src, deps):
            jobs.append(([NVCC] + NVFLAGS + ["-c", src, "-o", obj], obj))
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(OUT_DIR, f + ".o")
        if force or _stale(obj, src, deps):
            jobs.append((["g++"] + CXXFLAGS + ["-c", src, "-o", obj], obj))

    def run(job):
        cmd, obj = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r

    with ThreadPoolExecutor(max_workers=8) as ex:
        for obj, r in ex.map(run, jobs):
            if r.returncode != 0:
                raise RuntimeError(f"compile failed for {obj}:\n{r.stderr[-6000:]}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(obj + ".log", "w") as fh:
                fh.write(r.stderr)
    objs = [os.path.join(OUT_DIR, f + ".o") for f in CU + CPP]
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lpthread",
                                                                "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr[-6000:])
    return LIB


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
