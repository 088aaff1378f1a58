"""GPU unit tests of the tcgen05/TMA operand formats (self-test kernels in libfpdt.so) and of the
device twin of the input generator.  Reference = host matmul of the same bf16 values (fp64)."""
import ctypes

import numpy as np
import pytest
import torch

import fpdt_inputs as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2408_16978_b200 import _lib
    return _lib.load_diag()


@pytest.fixture(scope="module")
def genlib():
    from paper_2408_16978_b200 import _lib
    return _lib.load_generator()


def _rand_bf16(shape, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("d", [64, 80, 128])
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_umma_probe(lib, d, variant):
    H, rows = 3, 256
    b = _rand_bf16((rows, H, d), 1 + d).cuda()
    if variant == 0:
        a = _rand_bf16((rows, H, d), 2 + d).cuda()
        ref = a[:128, H - 1].double() @ b[:128, H - 1].double().T
        out = torch.empty(128, 128, dtype=torch.float32, device="cuda")
    else:
        a = _rand_bf16((128, 128), 3 + d).cuda()
        ref = a.double() @ b[:128, H - 1].double()
        out = torch.empty(128, d, dtype=torch.float32, device="cuda")
    rc = lib.fpdt_selftest_umma(variant, d, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), H, rows,
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(0))
    torch.cuda.synchronize()
    assert rc == 0
    err = (out.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("dist", gen.DISTRIBUTIONS)
@pytest.mark.parametrize("name", ["q", "k"])
def test_generator_device_twin_bitwise(genlib, dist, name):
    S, C, p, H, d = 1024, 256, 2, 4, 80
    for rank in range(p):
        s_local = S // p
        out = torch.empty(s_local, H, d, dtype=torch.bfloat16, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(out.data_ptr()), 0, gen.TENSOR_IDS[name], gen.DIST_IDS[dist], 11,
                                  s_local, H, d, S, rank, p, C, ctypes.c_void_p(0))
        torch.cuda.synchronize()
        assert rc == 0
        ref = gen.generate(name, dist, 11, gen.global_tokens_of_rank(rank, p, s_local, C), H, d, S)
        assert np.array_equal(out.float().cpu().numpy(), ref)
