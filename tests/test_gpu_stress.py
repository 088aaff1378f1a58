"""Scheduler stress (SURVEY §4 test tier 5): with FPDT_STRESS_NS set, the library puts a sleep kernel of random length
(up to that many ns) on the stream of every copy, all-to-all, projection GEMM and attention launch, before it.  The
streams then interleave in orders the unperturbed schedule never shows, so a missing cross-stream event edge (a fetch
that does not wait for its offload, a slot rewritten before its reader is done, an output read before its writer)
turns into wrong numbers.  Every schedule must stay bitwise equal to its unperturbed run for O, lse, dK, dV (their
arithmetic order is fixed) and within the reduce-order bound for dQ, and match the oracle."""
import os

import numpy as np
import pytest

import fpdt_inputs as gen
from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu

DQ_ORDER_TOL = 2.0 ** -8   # one bf16 rounding flip on the largest element (tests/test_gpu_bwd_order.py)


class stressed:
    """Contexts created inside read FPDT_STRESS_NS / FPDT_STRESS_SEED."""

    def __init__(self, ns=300000, seed=1):
        self.ns, self.seed = ns, seed

    def __enter__(self):
        os.environ["FPDT_STRESS_NS"] = str(self.ns)
        os.environ["FPDT_STRESS_SEED"] = str(self.seed)

    def __exit__(self, *exc):
        os.environ.pop("FPDT_STRESS_NS", None)
        os.environ.pop("FPDT_STRESS_SEED", None)


def _ctx(order=None, residency=None, keep=None):
    from paper_2408_16978_b200 import fpdt
    ctx = fpdt.FPDTContext()
    if order is not None:
        ctx.set_bwd_order(order)
    if residency is not None:
        ctx.set_residency(*residency)
    if keep is not None:
        ctx.set_sparsity(keep)
    return ctx


def _compare(got, base, ref, tol):
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), n
    assert rel_err(got["dq"], base["dq"]) < DQ_ORDER_TOL
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= tol for e in errs.values()), errs


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("case", ["kv_outer", "q_outer", "residency_sparse", "fp32"])
def test_stress_world1(case, seed):
    S, Hq, Hkv, d, C = 2048, 8, 2, 80, 256   # u = 8
    dtype = "fp32" if case == "fp32" else "bf16"
    if case == "fp32":
        S, d, C = 1024, 64, 256
    x = inputs("drift", 51, S, Hq, Hkv, d)
    kw = {}
    keep = None
    if case == "q_outer":
        kw = dict(order=1)
    elif case == "residency_sparse":
        keep = gen.sparsity_plan(S // C, 0.4, seed=11)
        kw = dict(residency=(2, 3), keep=keep)
    ctx = _ctx(**kw)
    base = run_cuda(x, C, dtype, 1, ctx=ctx)
    ctx.close()
    with stressed(seed=seed):
        ctx = _ctx(**kw)
        got = run_cuda(x, C, dtype, 1, ctx=ctx)
        ctx.close()
    assert base["stats"]["stress_sleeps"] == 0
    assert got["stats"]["stress_sleeps"] >= got["stats"]["attn_launches"]  # every launch (and copy) was perturbed
    if keep is None:
        ref = oracle_full(x)
    else:
        from oracle import attention
        o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
        dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"], keep=keep, chunk=C)
        ref = {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}
    _compare(got, base, ref, TOL[dtype])


@pytest.mark.parametrize("order", [0, 1])
def test_stress_multirank(order):
    """p = 2 through the local group: the per-chunk all-to-alls, the comm stream and the reverse exchanges."""
    from test_gpu_multirank import run_group
    S, Hq, Hkv, d, C = 2048, 8, 2, 128, 512
    x = gen.make_inputs("sink", 52, S, Hq, Hkv, d)
    base = run_group(x, 2, C, "bf16", 1, bwd_order=order)
    with stressed(seed=3):
        got = run_group(x, 2, C, "bf16", 1, bwd_order=order)
    _compare(got, base, oracle_full(x), TOL["bf16"])


def test_stress_block():
    """The fused-projection block at p = 2: projection GEMMs on the comm stream against the chunk pipeline."""
    from test_gpu_block import oracle_block, run_block
    S, hidden, Hq, Hkv, d, C = 1024, 256, 4, 2, 64, 256
    xin = gen.make_block_inputs("normal", 53, S, hidden, Hq, Hkv, d)
    op = gen.make_output_proj_inputs(53, S, hidden, Hq, d)
    base = run_block(xin, 2, C, "bf16", Hq, Hkv, d, oproj=op)
    with stressed(seed=4):
        got = run_block(xin, 2, C, "bf16", Hq, Hkv, d, oproj=op)
    for n in ("o", "lse", "y"):
        assert np.array_equal(got[n], base[n]), n
    for n in ("dx", "dw", "dwo"):
        assert rel_err(got[n], base[n]) < 1e-2, n
