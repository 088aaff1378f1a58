"""The production NCCL data plane on ONE GPU ("we perform the Alltoall", L365).

A world-size-1 context created WITH an NCCL id (include/fpdt.h fpdt_ctx_create) makes a one-rank communicator and
runs the sequence-parallel schedule: every chunk is packed, exchanged by ncclAlltoAll (the rank with itself) and
unpacked, and the outputs and gradients come back through the return all-to-alls -- the code path of world size > 1
with the real NCCL calls, which the in-process group (tests/test_gpu_multirank.py) replaces by copy-engine exchanges.
The results must equal the direct world-size-1 path (the caller's rows in place): O, lse, dK, dV bitwise (the same
kernels on the same values), dQ within its reduce order; and the oracle within the usual bound.  The exchange timing
proves the all-to-alls ran."""
import numpy as np
import pytest

from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu


def _ctx_nccl1():
    from paper_2408_16978_b200 import fpdt
    return fpdt.FPDTContext(1, 0, fpdt.fpdt_get_unique_id())


@pytest.mark.parametrize("dtype,d,Hq,Hkv,offload", [("bf16", 80, 2, 2, 1), ("bf16", 128, 4, 2, 1),
                                                    ("bf16", 80, 2, 2, 0), ("fp32", 64, 2, 2, 1)])
def test_one_rank_nccl_exchange_path(dtype, d, Hq, Hkv, offload):
    S, C = 2048, 512
    x = inputs("drift", 5, S, Hq, Hkv, d)
    ctx = _ctx_nccl1()
    ctx.set_kernel_timing(True)
    got = run_cuda(x, C, dtype, offload, ctx=ctx)
    n_xch = ctx.exchange_time()["n"]
    ctx.close()
    ref = run_cuda(x, C, dtype, offload)
    # 4 chunks: forward 4 exchanges + 4 returns, backward 4 (O, dO) exchanges + 4 returns of (dq, dk, dv) at least
    assert n_xch >= 16, n_xch
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], ref[n]), n
    assert rel_err(got["dq"], ref["dq"]) < (1e-2 if dtype == "bf16" else 1e-5)
    exact = oracle_full(x)
    errs = {n: rel_err(got[n], exact[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL[dtype] for e in errs.values()), errs


def test_one_rank_nccl_host_io_and_q_outer():
    """The same path with the caller's tensors in pinned host memory and the GQA-aware Q-outer backward."""
    from paper_2408_16978_b200 import fpdt
    S, C, d = 2048, 512, 128
    x = inputs("normal", 6, S, 8, 2, d)
    ctx = _ctx_nccl1()
    ctx.set_bwd_order(fpdt.FPDT_BWD_Q_OUTER)
    got = run_cuda(x, C, "bf16", 1, ctx=ctx, host_io=True)
    ctx.close()
    exact = oracle_full(x)
    errs = {n: rel_err(got[n], exact[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
