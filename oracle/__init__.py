"""TEST INFRASTRUCTURE ONLY — the checkers for the CUDA hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline; the product package (paper_1504_04804_b200) never
imports it.

* :mod:`oracle.seq`  — ctypes binding of ``_ref/libmgoracle.so``, the plain-C
  restatement of the reference's sequential oracles (seq_oracle.c, citing
  /root/reference/proj/core/src/reference.cpp line by line).
* :mod:`oracle.ref`  — ctypes binding of ``_ref/libmgraph_ref.so``, the
  unmodified reference core compiled from /root/reference by oracle/Makefile
  plus the extern "C" shim ref_shim.cpp.  Parity is pinned against it and
  against the golden vectors in tests/golden/.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def build(quiet=True):
    """Compile the checkers (restatement always; reference when present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)
