"""GPU leg of the exhaustive libm sweep: the device glibc expf restatement
(csrc/glibc_expf.h, compiled by nvcc for sm_100a) and the exact-mode SiLU
x / (1 + expf(-x)) (proj/src/eltwise.cpp:31-34) over ALL 2^32 float bit
patterns, against the live host libm of the box (the build glibc's ifunc
dispatches to, which the library probes at load time)."""
import ctypes as C
import pathlib
import subprocess

import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]
CHUNK = 1 << 28  # 1 GiB of fp32 results per device pass


@pytest.fixture(scope="module")
def host_check(tmp_path_factory):
    so = tmp_path_factory.mktemp("expf") / "libexpf_check.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-pthread", "-shared", "-fPIC",
                    str(ROOT / "tests" / "native" / "expf_check.cpp"), "-o", str(so)], check=True)
    lib = C.CDLL(str(so))
    lib.expf_check.restype = C.c_ulonglong
    lib.expf_check.argtypes = [C.c_void_p, C.c_uint32, C.c_ulonglong, C.c_int, C.POINTER(C.c_ulonglong)]
    return lib


@pytest.mark.parametrize("mode", [0, 1], ids=["expf", "silu"])
def test_device_expf_all_inputs(host_check, mode):
    L = sb._lib()
    L.sige_debug_expf_sweep.restype = C.c_int
    L.sige_debug_expf_sweep.argtypes = [C.c_uint32, C.c_longlong, C.c_int, C.c_void_p, C.c_void_p]
    dev = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    host = torch.empty(CHUNK, dtype=torch.float32).pin_memory()
    total = 0
    for first in range(0, 1 << 32, CHUNK):
        assert L.sige_debug_expf_sweep(first, CHUNK, mode, dev.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream) == 0
        host.copy_(dev)
        torch.cuda.synchronize()
        where = C.c_ulonglong(0)
        bad = host_check.expf_check(host.data_ptr(), first, CHUNK, mode, C.byref(where))
        assert bad == 0, (f"{bad} mismatches in [{first:#x}, +{CHUNK:#x}); first at bits "
                          f"{first + where.value:#010x} (host fma build: {L.sige_debug_host_expf_is_fma()})")
        total += CHUNK
    assert total == 1 << 32
