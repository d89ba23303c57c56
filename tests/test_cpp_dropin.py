"""C++ drop-in: the reference's own unit tests for the host API it exports
(tests/test_cache.cpp, test_plan.cpp, test_minibatch.cpp, test_timing.cpp —
43 cases, ~31k checks) compiled UNMODIFIED against include/hybridsim/*.hpp and
linked to libhybridcache_b200.so instead of the reference library
(examples/reference_tests/Makefile). Host bookkeeping only: no GPU needed.
Needs the reference sources, so it runs in the build container only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/tests"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources absent (GPU box)")
def test_reference_unit_tests_pass_against_the_dropin_headers():
    mk = os.path.join(ROOT, "examples", "reference_tests")
    r = subprocess.run(["make", "-s", "-C", mk, "-j4", "run"], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    summary = [ln for ln in out.splitlines() if "test cases:" in ln][-1]
    assert "0 failed" in summary and "43 passed" in summary, summary
    # the binary links the product library, not the reference's
    ldd = subprocess.run(["ldd", os.path.join(ROOT, "build", "reference_tests", "dropin_tests")],
                         capture_output=True, text=True).stdout
    assert "libhybridcache_b200.so" in ldd and "hybridsim_ref" not in ldd
