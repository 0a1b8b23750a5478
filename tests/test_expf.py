"""The device SiLU's expf restatement (csrc/glibc_expf.h) against the live
host libm over ALL 2^32 float inputs (compiled as host code), for the libm
build this host dispatches to, and the SSE2 build with FMA masked off.
(The GPU leg of the same sweep is in tests/test_gpu_expf.py.)"""
import os
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def sweep_bin(tmp_path_factory):
    out = tmp_path_factory.mktemp("expf") / "expf_sweep"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-pthread",
                    f"-I{ROOT / 'paper_2211_02048_b200' / 'csrc'}", str(ROOT / "tests" / "native" / "expf_sweep.cpp"),
                    "-o", str(out)], check=True)
    return out


def _fma_host() -> bool:
    flags = pathlib.Path("/proc/cpuinfo").read_text()
    return " fma " in flags and " avx2 " in flags


def test_expf_exhaustive_default_variant(sweep_bin):
    r = subprocess.run([str(sweep_bin), "1" if _fma_host() else "0"], capture_output=True, text=True)
    assert r.returncode == 0 and "mismatches 0" in r.stdout, r.stdout + r.stderr


def test_expf_exhaustive_sse2_variant(sweep_bin):
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2_Usable,-FMA_Usable,-AVX2,-FMA")
    r = subprocess.run([str(sweep_bin), "0"], capture_output=True, text=True, env=env)
    assert r.returncode == 0 and "mismatches 0" in r.stdout, r.stdout + r.stderr
