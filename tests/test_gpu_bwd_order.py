"""GQA-aware Q-outer backward (include/fpdt.h fpdt_set_bwd_order).

The paper's backward (fig:bw_db) runs key/value chunks in the outer loop and streams the fp32 dq
partials of the query chunks through host memory.  The Q-outer order runs query chunks in the outer loop and streams
the fp32 dK/dV partials instead.  Both compute the same sums (§8(c) c.1) with the same pair kernels, and dK_j/dV_j
accumulate over query chunks i = j, j+1, ... in the same order in both, so O, lse, dK, dV are bitwise equal to the
paper order's; dQ equal up to the order of its fp32 reduce-adds; all match the oracle.  The host bytes follow each
schedule exactly (counted here independently of the library's own AUTO model)."""
import numpy as np
import pytest

import fpdt_inputs as gen
from fpdt_testlib import TOL, expected_bwd_bytes, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu

KV_OUTER, Q_OUTER, AUTO = 0, 1, 2
# dQ of the two orders: the same fp32 sums in a different reduce-add order, then bf16 RNE; one rounding flip on the
# largest element is 2^-8 of the max (normwise), so the bound is that ulp
DQ_ORDER_TOL = 2.0 ** -8


def run_order(x, C, dtype, order, keep=None, residency=None):
    from paper_2408_16978_b200 import fpdt
    ctx = fpdt.FPDTContext()
    if keep is not None:
        ctx.set_sparsity(keep)
    if residency is not None:
        ctx.set_residency(*residency)
    ctx.set_bwd_order(order)
    # forward alone first, to separate the backward's host bytes
    fwd = run_cuda(x, C, dtype, 1, ctx=ctx, want_grad=False)["stats"]
    got = run_cuda(x, C, dtype, 1, ctx=ctx)
    ctx.close()
    s1 = got["stats"]
    got["bwd_h2d"] = s1["bytes_h2d"] - 2 * fwd["bytes_h2d"]
    got["bwd_d2h"] = s1["bytes_d2h"] - 2 * fwd["bytes_d2h"]
    return got


@pytest.mark.parametrize("d,Hq,Hkv", [(80, 4, 4), (128, 8, 2), (64, 8, 1)])
def test_q_outer_matches_paper_order(d, Hq, Hkv):
    S, C = 2048, 512   # u = 4
    u = S // C
    x = inputs("drift", 31, S, Hq, Hkv, d)
    base = run_order(x, C, "bf16", KV_OUTER)
    got = run_order(x, C, "bf16", Q_OUTER)
    assert got["stats"]["bwd_order"] == Q_OUTER and base["stats"]["bwd_order"] == KV_OUTER
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), n
    assert rel_err(got["dq"], base["dq"]) < DQ_ORDER_TOL
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    do_off = S * Hq * d * 2   # the preamble's dO offload (both orders)
    for r, order in ((got, Q_OUTER), (base, KV_OUTER)):
        h2d, d2h = expected_bwd_bytes(order, u, C, Hq, Hkv, d, 2)
        assert (r["bwd_h2d"], r["bwd_d2h"]) == (h2d, d2h + do_off), order


def test_q_outer_fp32():
    S, Hq, Hkv, d, C = 1024, 4, 2, 64, 256   # u = 4, fp32 validation mode
    x = inputs("peaky", 32, S, Hq, Hkv, d)
    got = run_order(x, C, "fp32", Q_OUTER)
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["fp32"] for e in errs.values()), errs


@pytest.mark.parametrize("Hq,Hkv,want", [(4, 4, KV_OUTER), (8, 2, Q_OUTER), (8, 1, Q_OUTER)])
def test_auto_picks_fewer_host_bytes(Hq, Hkv, want):
    S, d, C = 2048, 128, 256   # u = 8
    u = S // C
    x = inputs("normal", 33, S, Hq, Hkv, d)
    got = run_order(x, C, "bf16", AUTO)
    assert got["stats"]["bwd_order"] == want
    kvo = sum(expected_bwd_bytes(KV_OUTER, u, C, Hq, Hkv, d, 2))
    qo = sum(expected_bwd_bytes(Q_OUTER, u, C, Hq, Hkv, d, 2))
    assert (qo < kvo) == (want == Q_OUTER)
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


@pytest.mark.parametrize("residency", [None, (2, 3), (8, 8)])
def test_q_outer_sparse_and_resident(residency):
    """Q-outer composes with a block-sparsity plan (dK_j/dV_j final at the last query chunk keeping j) and the
    residency budget (resident key/value chunks keep their dK/dV partial on the device)."""
    from oracle import attention
    S, Hq, Hkv, d, C = 2048, 8, 2, 80, 256   # u = 8
    u = S // C
    keep = gen.sparsity_plan(u, 0.4, seed=7)
    x = inputs("sink", 34, S, Hq, Hkv, d)
    base = run_order(x, C, "bf16", KV_OUTER, keep=keep, residency=residency)
    got = run_order(x, C, "bf16", Q_OUTER, keep=keep, residency=residency)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), n
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"], keep=keep, chunk=C)
    ref = {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    rkv, rq = residency or (0, 0)
    rq_eff = min(rq, u)
    do_off = sum(C * Hq * d * 2 for i in range(u) if not i >= u - rq_eff)
    h2d, d2h = expected_bwd_bytes(Q_OUTER, u, C, Hq, Hkv, d, 2, keep=keep, rkv=min(rkv, u), rq=rq_eff)
    assert (got["bwd_h2d"], got["bwd_d2h"]) == (h2d, d2h + do_off)


@pytest.mark.parametrize("p,Hq,Hkv", [(2, 8, 2), (4, 8, 4), (8, 16, 8)])
def test_q_outer_multirank(p, Hq, Hkv):
    """p > 1 through the local group: dq_i and (dk_j, dv_j) return by separate all-to-alls; world-size invariance
    against the p = 1 paper-order run (bitwise for O, lse, dK, dV) and oracle parity."""
    from test_gpu_multirank import run_group
    S, d, C = 2048 * max(1, p // 4), 128, 512 * max(1, p // 4)   # p = 8: the 70B shape, one kv head per rank
    x = gen.make_inputs("drift", 35, S, Hq, Hkv, d)
    base = run_group(x, 1, C, "bf16", 1)
    stats = {}
    got = run_group(x, p, C, "bf16", 1, bwd_order=Q_OUTER, stats=stats)
    assert all(s["bwd_order"] == Q_OUTER for s in stats.values())
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), n
    assert rel_err(got["dq"], base["dq"]) < DQ_ORDER_TOL
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_bad_order_rejected():
    from paper_2408_16978_b200 import fpdt
    ctx = fpdt.FPDTContext()
    with pytest.raises(fpdt.FpdtError):
        ctx.set_bwd_order(7)
    ctx.close()
