"""HBM residency budget (include/fpdt.h fpdt_set_residency) at world size 1.

Resident key/value chunks (i < kv_chunks) and query-side chunks (i >= u - q_chunks) are read in place instead of
being offloaded and fetched.  The arithmetic is the offloaded schedule's: O, lse, dK, dV are bitwise equal to the
fully offloaded run, dQ equal up to the order of its fp32 reduce-adds; both match the oracle.  The host-to-device
bytes follow the schedule exactly (PAPER.md L230, L365 with the resident chunks' fetches removed)."""
import numpy as np
import pytest

from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu


def expected_h2d(u, C, Hq, Hkv, d, eb, rkv, rq):
    kv = C * 2 * Hkv * d * eb
    qc = C * Hq * d * eb
    dqc = C * Hq * d * 4
    kres = lambda i: i < min(rkv, u)
    qres = lambda i: i >= u - min(rq, u)
    fwd = sum(kv for m in range(u) for i in range(m) if not kres(i))
    bwd = sum(kv for j in range(u) if not kres(j))
    bwd += sum(2 * qc for j in range(u) for i in range(j, u) if not qres(i))
    bwd += sum(dqc for j in range(1, u) for i in range(j, u) if not qres(i))
    return fwd + bwd


@pytest.mark.parametrize("d,Hq,Hkv", [(80, 4, 4), (128, 8, 2)])
@pytest.mark.parametrize("residency", [(1, 1), (2, 3), (0, 4), (4, 0), (8, 8)])
def test_residency_p1(d, Hq, Hkv, residency):
    from paper_2408_16978_b200 import fpdt
    S, C = 2048, 512   # u = 4
    u = S // C
    x = inputs("drift", 21, S, Hq, Hkv, d)
    base = run_cuda(x, C, "bf16", 1)
    ctx = fpdt.FPDTContext()
    ctx.set_residency(*residency)
    got = run_cuda(x, C, "bf16", 1, ctx=ctx)
    ctx.close()
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), (n, residency)
    assert rel_err(got["dq"], base["dq"]) < 1e-3
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    assert got["stats"]["bytes_h2d"] == expected_h2d(u, C, Hq, Hkv, d, 2, *residency)
    assert base["stats"]["bytes_h2d"] == expected_h2d(u, C, Hq, Hkv, d, 2, 0, 0)


def test_residency_with_sparsity():
    """The residency budget composes with a block-sparsity plan (dropped blocks stay dropped)."""
    import fpdt_inputs as gen
    from oracle import attention
    from paper_2408_16978_b200 import fpdt
    S, Hq, Hkv, d, C = 2048, 4, 2, 64, 256   # u = 8
    keep = gen.sparsity_plan(S // C, 0.4, seed=5)
    x = inputs("normal", 22, S, Hq, Hkv, d)
    ctx = fpdt.FPDTContext()
    ctx.set_sparsity(keep)
    ctx.set_residency(3, 2)
    got = run_cuda(x, C, "bf16", 1, ctx=ctx)
    ctx.close()
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"], keep=keep, chunk=C)
    ref = {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
