"""GPU tests of the conv kernel's alternative code paths, each selected by an
environment switch the library reads once per process — so each runs the
integer bit-exact and tolerance suites of test_gpu_tc.py in a subprocess:

* SIGE_FORCE_SPLITK=8: every static-count launch split over a thread-block
  cluster (DSMEM reduce-scatter) — exact integer sums pin the reduction.
* SIGE_NO_TMA_A=1: A windows staged by the per-thread cp.async ring instead
  of 128-byte-swizzled TMA boxes.
* SIGE_NO_TUNE=1 / SIGE_NO_SPLITK=1: the analytic plan without split-K.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"SIGE_FORCE_SPLITK": "8"}, {"SIGE_NO_TMA_A": "1"},
                                 {"SIGE_NO_TUNE": "1", "SIGE_NO_SPLITK": "1"}],
                         ids=["splitk8", "cp_async_a", "analytic_nosplit"])
def test_tc_suite_under_variant(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_tc.py")],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
