"""Host-memory calls (include/fpdt.h fpdt_attn_fwd_host / fpdt_attn_bwd_host): the caller's q, k, v, o, lse, dO, dq,
dk, dv live in pinned host memory and the library stages them chunk by chunk inside its own copy schedule (the paper
keeps activations in host memory and brings each chunk to the GPU when needed).

The staging only changes where rows come from and go to, not the arithmetic: O, lse, dK, dV must be bitwise equal to
the device-memory calls on the same inputs (dQ within its reduce order), at world size 1 (where q_i and dO_i are
fetched straight from the caller's rows and D_i is formed at the first pair of query chunk i) and through the
in-process group at world sizes 2 and 4, with a sparsity plan, under scheduler stress, and against the fp64 oracle.
The byte counters show what moved: each caller row once in each direction."""
import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu

DQ_ORDER_TOL = 2.0 ** -8


def _same(got, base):
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), (n, rel_err(got[n], base[n]))
    assert rel_err(got["dq"], base["dq"]) < DQ_ORDER_TOL


@pytest.mark.parametrize("dtype,d", [("bf16", 64), ("bf16", 80), ("bf16", 128), ("fp32", 80)])
def test_host_io_world1(dtype, d):
    S, Hq, Hkv, C = (2048, 8, 2, 512) if dtype == "bf16" else (1024, 4, 2, 256)
    x = inputs("drift", 71, S, Hq, Hkv, d)
    base = run_cuda(x, C, dtype, 1)
    got = run_cuda(x, C, dtype, 1, host_io=True)
    _same(got, base)
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL[dtype] for e in errs.values()), errs
    st, sb = got["stats"], base["stats"]
    eb = 2 if dtype == "bf16" else 4
    bq, bkv = S * Hq * d * eb, S * Hkv * d * eb
    # world size 1: q, k, v uploaded once; dO_i and q_i fetched from the caller's rows by the chunk loop (counted
    # there), so nothing else of the caller's is uploaded
    assert st["bytes_io_h2d"] == bq + 2 * bkv
    assert st["bytes_io_d2h"] == bq + S * Hq * 4 + bq + 2 * bkv   # o, lse, dq, dk, dv
    # the device path offloads q and dO (2 * bq) that the host path reads in place
    assert sb["bytes_d2h"] - st["bytes_d2h"] == 2 * bq
    assert st["bytes_h2d"] == sb["bytes_h2d"]
    assert sb["bytes_io_h2d"] == 0 and sb["bytes_io_d2h"] == 0


def test_host_io_world1_sparse_and_no_lse():
    from paper_2408_16978_b200 import fpdt
    S, Hq, Hkv, d, C = 2048, 8, 4, 80, 256       # u = 8
    x = inputs("sink", 72, S, Hq, Hkv, d)
    keep = gen.sparsity_plan(S // C, 0.5, seed=3)
    res = []
    for host in (False, True):
        ctx = fpdt.FPDTContext()
        ctx.set_sparsity(keep)
        res.append(run_cuda(x, C, "bf16", 1, ctx=ctx, host_io=host))
        ctx.close()
    _same(res[1], res[0])
    # lse = NULL, forward only
    q, k, v = (torch.tensor(x[n]).to(torch.bfloat16).pin_memory() for n in ("q", "k", "v"))
    o = torch.empty_like(q).pin_memory()
    ctx = fpdt.FPDTContext()
    fpdt.fpdt_attn_fwd_host(ctx, q, k, v, o, None, S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    ctx.close()
    ref = run_cuda(x, C, "bf16", 1, want_grad=False)
    assert np.array_equal(o.float().numpy(), ref["o"])


def test_host_io_other_o_buffer():
    """The backward's o argument need not be the forward's output buffer (then it is uploaded first)."""
    from paper_2408_16978_b200 import fpdt
    S, Hq, Hkv, d, C = 1024, 4, 4, 64, 256
    x = inputs("normal", 73, S, Hq, Hkv, d)
    base = run_cuda(x, C, "bf16", 1)
    q, k, v, do = (torch.tensor(x[n]).to(torch.bfloat16).pin_memory() for n in ("q", "k", "v", "do"))
    o = torch.empty_like(q).pin_memory()
    lse = torch.empty(S, Hq, dtype=torch.float32).pin_memory()
    ctx = fpdt.FPDTContext()
    fpdt.fpdt_attn_fwd_host(ctx, q, k, v, o, lse, S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    o2 = o.clone().pin_memory()
    o.zero_()  # the forward's buffer no longer holds the output
    dq, dk, dv = (torch.empty_like(t).pin_memory() for t in (q, k, v))
    before = ctx.stats()["bytes_io_h2d"]
    fpdt.fpdt_attn_bwd_host(ctx, o2, do, dq, dk, dv, S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    assert ctx.stats()["bytes_io_h2d"] - before == S * Hq * d * 2   # o uploaded
    ctx.close()
    got = {"o": o2.float().numpy(), "lse": lse.numpy(), "dq": dq.float().numpy(), "dk": dk.float().numpy(),
           "dv": dv.float().numpy()}
    _same(got, base)


@pytest.mark.parametrize("p", [2, 4])
def test_host_io_multirank(p):
    from test_gpu_multirank import run_group
    S, Hq, Hkv, d, C = 2048, 8, 4, 80, 512
    x = gen.make_inputs("drift", 74, S, Hq, Hkv, d)
    stats = {}
    got = run_group(x, p, C, "bf16", 1, host_io=True, stats=stats)
    base = run_group(x, p, C, "bf16", 1)
    _same(got, base)
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    s_local = S // p
    bq, bkv = s_local * Hq * d * 2, s_local * Hkv * d * 2
    for r in range(p):
        assert stats[r]["bytes_io_h2d"] == bq + 2 * bkv + bq       # q, k, v, dO
        assert stats[r]["bytes_io_d2h"] == bq + s_local * Hq * 4 + bq + 2 * bkv


def test_host_io_multirank_leader_fetch():
    from test_gpu_multirank import run_group
    S, Hq, Hkv, d, C = 2048, 8, 2, 64, 512
    x = gen.make_inputs("normal", 75, S, Hq, Hkv, d)
    got = run_group(x, 2, C, "bf16", 1, host_io=True, fetch=1)
    base = run_group(x, 2, C, "bf16", 1)
    _same(got, base)


@pytest.mark.parametrize("seed", [1, 2])
def test_host_io_stress(seed):
    from test_gpu_stress import stressed
    from paper_2408_16978_b200 import fpdt
    S, Hq, Hkv, d, C = 2048, 8, 2, 80, 256   # u = 8
    x = inputs("drift", 76, S, Hq, Hkv, d)
    base = run_cuda(x, C, "bf16", 1, host_io=True)
    with stressed(seed=seed):
        ctx = fpdt.FPDTContext()
        got = run_cuda(x, C, "bf16", 1, ctx=ctx, host_io=True)
        ctx.close()
    assert got["stats"]["stress_sleeps"] >= got["stats"]["attn_launches"]
    _same(got, base)


def test_host_io_stress_multirank():
    from test_gpu_multirank import run_group
    from test_gpu_stress import stressed
    S, Hq, Hkv, d, C = 2048, 8, 4, 80, 512
    x = gen.make_inputs("drift", 77, S, Hq, Hkv, d)
    base = run_group(x, 2, C, "bf16", 1, host_io=True)
    with stressed(seed=3):
        got = run_group(x, 2, C, "bf16", 1, host_io=True)
    _same(got, base)


def test_host_io_errors():
    from paper_2408_16978_b200 import fpdt
    S, Hq, Hkv, d, C = 1024, 4, 4, 64, 256
    x = inputs("normal", 78, S, Hq, Hkv, d)
    hq, hk, hv, hdo = (torch.tensor(x[n]).to(torch.bfloat16).pin_memory() for n in ("q", "k", "v", "do"))
    ho = torch.empty_like(hq).pin_memory()
    dq, dk, dv = (torch.empty_like(t).pin_memory() for t in (hq, hk, hv))
    dev = {n: t.cuda() for n, t in (("q", hq), ("k", hk), ("v", hv), ("do", hdo))}
    do_ = torch.empty_like(dev["q"])
    args = (S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16)

    def code_of(fn, *a):
        with pytest.raises(fpdt.FpdtError) as e:
            fn(*a)
        return e.value.code

    ctx = fpdt.FPDTContext()
    assert code_of(fpdt.fpdt_attn_fwd_host, ctx, hq, hk, hv, ho, None, *args, 0) == fpdt.FPDT_ERR_UNSUPPORTED
    ctx.set_residency(1, 0)
    assert code_of(fpdt.fpdt_attn_fwd_host, ctx, hq, hk, hv, ho, None, *args, 1) == fpdt.FPDT_ERR_UNSUPPORTED
    ctx.set_residency(0, 0)
    fpdt.fpdt_attn_fwd_host(ctx, hq, hk, hv, ho, None, *args, 1)
    torch.cuda.synchronize()
    # host forward -> device backward, and device forward -> host backward, are refused
    assert code_of(fpdt.fpdt_attn_bwd, ctx, dev["q"], dev["do"], do_, do_, do_, *args, 1) == fpdt.FPDT_ERR_STATE
    fpdt.fpdt_attn_fwd(ctx, dev["q"], dev["k"], dev["v"], do_, None, *args, 1)
    torch.cuda.synchronize()
    assert code_of(fpdt.fpdt_attn_bwd_host, ctx, ho, hdo, dq, dk, dv, *args, 1) == fpdt.FPDT_ERR_STATE
    ctx.close()
