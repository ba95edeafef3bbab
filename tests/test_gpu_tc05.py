"""tcgen05 kind::tf32 building block (libdgm_probe.so): descriptors, TMEM, 3xTF32 accuracy."""

import ctypes
import os

import numpy as np
import pytest
from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PROBE = os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so")


@pytest.fixture(scope="module")
def probe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = ctypes.CDLL(PROBE)
    lib.dgm_probe_tf32_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    lib.dgm_probe_tf32_gemm_ts.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("n,k", [(40, 40), (48, 64), (256, 8), (8, 16), (112, 40)])
def test_tf32_and_3xtf32_gemm(probe, n, k):
    gen = torch.Generator(device="cuda").manual_seed(n * 100 + k)
    a = torch.randn(128, k, device="cuda", generator=gen)
    b = torch.randn(n, k, device="cuda", generator=gen)
    want = (a.double() @ b.double().T)
    errs = {}
    for passes in (1, 3):
        c = torch.full((128, n), float("nan"), device="cuda")
        rc = probe.dgm_probe_tf32_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, k, passes,
                                       torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        errs[passes] = ((c.double() - want).norm() / want.norm()).item()
    print(f"n={n} k={k} tf32 {errs[1]:.2e} 3xtf32 {errs[3]:.2e}")
    assert errs[1] < 5e-3          # plain TF32: ~2^-11 per product
    assert errs[3] < 2e-6          # 3xTF32: fp32-class accuracy
    assert errs[3] < errs[1] / 50


@pytest.mark.parametrize("n,k", [(48, 64), (16, 8), (32, 40), (256, 16)])
def test_tf32_gemm_a_in_tmem(probe, n, k):
    """TS form: A written to TMEM with tcgen05.st (lane = row), B from smem."""
    gen = torch.Generator(device="cuda").manual_seed(n + k)
    a = torch.randn(128, k, device="cuda", generator=gen)
    b = torch.randn(n, k, device="cuda", generator=gen)
    want = (a.double() @ b.double().T)
    errs = {}
    for passes in (1, 3):
        c = torch.full((128, n), float("nan"), device="cuda")
        rc = probe.dgm_probe_tf32_gemm_ts(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, k, passes,
                                          torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        errs[passes] = ((c.double() - want).norm() / want.norm()).item()
    print(f"TS n={n} k={k} tf32 {errs[1]:.2e} 3xtf32 {errs[3]:.2e}")
    assert errs[1] < 5e-3 and errs[3] < 2e-6


def test_tf32_inputs_are_truncated(probe):
    """kind::tf32 reads fp32 operands and drops the low 13 mantissa bits (round toward zero).

    The v2 stage kernel feeds the raw state rows as the 'hi' operand of its 3xTF32 volume product
    and splits only lo = x - trunc(x); that is exact only if the hardware truncates.  Passes=13 makes
    the probe store the hi operands unmasked: the error must stay at the masked 3xTF32 level.
    """
    gen = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn(128, 40, device="cuda", generator=gen)
    b = torch.randn(112, 40, device="cuda", generator=gen)
    want = (a.double() @ b.double().T)
    errs = {}
    for passes in (3, 13):
        c = torch.full((128, 112), float("nan"), device="cuda")
        assert probe.dgm_probe_tf32_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), 112, 40, passes,
                                         torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        errs[passes] = ((c.double() - want).norm() / want.norm()).item()
    print(f"3xtf32 masked {errs[3]:.2e} raw {errs[13]:.2e}")
    assert errs[13] < 2e-6
