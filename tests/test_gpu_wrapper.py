"""GPU: the C++ drop-in (include/mdvec_gpu.hpp) with the reference's own types
and error taxonomy, checked against the reference's own kernels by
oracle/_ref/wrapper_check (built in the build container where the reference
headers exist; see oracle/Makefile `wrapper`)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference_kernels():
    exe = os.path.join(ROOT, "oracle", "_ref", "wrapper_check")
    if not os.path.exists(exe):
        pytest.skip("wrapper_check not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[FAIL]" not in r.stdout
    assert r.stdout.count("[PASS]") >= 80
