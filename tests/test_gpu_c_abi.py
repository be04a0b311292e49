"""The boundary exercised from outside Python, on the GPU:

* tests/c/lgs_c_demo.c -- a plain C99 program linked with liblgs.so (built by build()): three of the
  reference's renderer tests through the C ABI;
* oracle/_ref/shim_vs_reference -- the C++ drop-in include/legoslam_gpu.hpp, called with the exact
  lego::render / lego::render_backward signatures, against the reference's own renderer.cpp in the
  same program (built by oracle/Makefile where /root/reference exists; skipped where it was not)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(path):
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    return r


def test_c_program_against_the_abi():
    exe = os.path.join(ROOT, "tests", "c", "build", "lgs_c_demo")
    if not os.path.exists(exe):
        pytest.fail("tests/c/build/lgs_c_demo missing: run __graft_entry__.build()")
    r = _run(exe)
    assert r.returncode == 0 and "0 failure(s)" in r.stdout


def test_cpp_drop_in_against_the_reference():
    exe = os.path.join(ROOT, "oracle", "_ref", "shim_vs_reference")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/shim_vs_reference not built (needs /root/reference at build time)")
    r = _run(exe)
    assert r.returncode == 0 and "0 failure(s)" in r.stdout
