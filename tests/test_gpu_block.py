"""Attention block with the fused chunked QKV projection (include/fpdt.h fpdt_block_fwd / fpdt_block_bwd;
SURVEY §8(f) NEXT-3) against oracle/block.py (fp64): O, lse, the hidden-state gradient dx
and the weight gradient dW, normwise max relative error <= 1e-2 (bf16) / 1e-4 (fp32); p = 1 and, through the
single-GPU local group, p = 2 and 4 (dW summed over ranks, as a data-parallel all-reduce would)."""
import threading

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, rel_err
from oracle import attention, block

pytestmark = pytest.mark.gpu


def run_block(xin: dict, p: int, C: int, dtype: str, Hq: int, Hkv: int, d: int, keep=None, oproj=None,
              hidden_offload=False, stats=None, nccl1=False) -> dict:
    """oproj: {"wo", "dy"} for the output projection (y = o wo; the backward starts from dy).  hidden_offload: the
    forward offloads x and the backward gets x = None (fpdt_set_hidden_offload).  nccl1: world size 1 through a one-rank
    NCCL communicator (the exchange path, tests/test_gpu_nccl.py)."""
    from paper_2408_16978_b200 import fpdt
    S, hidden = xin["x"].shape
    s_local = S // p
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = fpdt.dtype_code(tdt)
    group = fpdt.LocalGroup(p) if p > 1 else None
    rows = [gen.global_tokens_of_rank(r, p, s_local, C) for r in range(p)]
    out = {"o": np.zeros((S, Hq, d), np.float32), "lse": np.zeros((S, Hq), np.float32),
           "dx": np.zeros((S, hidden), np.float32), "dw": [None] * p, "y": np.zeros((S, hidden), np.float32),
           "dwo": [None] * p}
    errors = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                x = torch.tensor(xin["x"][rows[r]]).to(tdt).cuda().contiguous()
                w = torch.tensor(xin["w"]).to(tdt).cuda().contiguous()
                do = torch.tensor(xin["do"][rows[r]]).to(tdt).cuda().contiguous()
                wo = y = dwo = None
                if oproj is not None:
                    wo = torch.tensor(oproj["wo"]).to(tdt).cuda().contiguous()
                    do = torch.tensor(oproj["dy"][rows[r]]).to(tdt).cuda().contiguous()   # dL/dy
                    y = torch.empty(s_local, hidden, dtype=tdt, device="cuda")
                    dwo = torch.full(tuple(wo.shape), float("nan"), dtype=torch.float32, device="cuda")
                o = torch.empty(s_local, Hq, d, dtype=tdt, device="cuda")
                lse = torch.empty(s_local, Hq, dtype=torch.float32, device="cuda")
                dx = torch.empty_like(x)
                dw = torch.full(tuple(w.shape), float("nan"), dtype=torch.float32, device="cuda")
            stream.synchronize()
            if p > 1:
                ctx = fpdt.FPDTContext(p, r, group=group)
            else:
                ctx = fpdt.FPDTContext(1, 0, fpdt.fpdt_get_unique_id()) if nccl1 else fpdt.FPDTContext()
            if keep is not None:
                ctx.set_sparsity(keep)
            if hidden_offload:
                ctx.set_hidden_offload(True)
            fpdt.fpdt_block_fwd(ctx, x, w, o, lse, s_local, hidden, Hq, Hkv, d, 1, C, p, code, 1, 0.0, stream,
                                w_o=wo, y=y)
            fpdt.fpdt_block_bwd(ctx, None if hidden_offload else x, w, o, do, dx, dw, s_local, hidden, Hq, Hkv, d, 1, C,
                                p, code, 1, 0.0, stream, w_o=wo, dw_o=dwo)
            stream.synchronize()
            out["o"][rows[r]] = o.float().cpu().numpy()
            out["lse"][rows[r]] = lse.cpu().numpy()
            out["dx"][rows[r]] = dx.float().cpu().numpy()
            out["dw"][r] = dw.cpu().numpy()
            if stats is not None:
                stats[r] = ctx.stats()
            if oproj is not None:
                out["y"][rows[r]] = y.float().cpu().numpy()
                out["dwo"][r] = dwo.cpu().numpy()
            ctx.close()
        except Exception as e:  # surfaced in the main thread
            errors.append((r, e))

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(p)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "a rank hung"
    if group is not None:
        group.close()
    assert not errors, errors
    out["dw"] = np.sum(out["dw"], axis=0)
    out["dwo"] = np.sum(out["dwo"], axis=0) if oproj is not None else None
    return out


def oracle_block(xin, Hq, Hkv, d, dtype, keep=None, C=0):
    """bf16 mode: q, k, v and dq, dk, dv are bf16 tensors (reading R27, oracle/block.py)."""
    r = dtype == "bf16"
    dx, dw = block.block_backward(xin["x"], xin["w"], xin["do"], Hq, Hkv, d, bf16_intermediates=r, keep=keep,
                                  chunk=C)
    q, k, v = block.split_qkv(block._project(xin["x"], xin["w"], r), Hq, Hkv, d)
    o, lse = attention.attention_forward(q, k, v, keep=keep, chunk=C)
    return {"o": o, "lse": lse, "dx": dx, "dw": dw}


@pytest.mark.parametrize("p,S,hidden,Hq,Hkv,d,C", [
    (1, 2048, 256, 4, 2, 64, 512),
    (1, 2048, 320, 4, 4, 80, 512),
    (1, 1024, 256, 8, 2, 128, 256),
    (2, 2048, 256, 4, 2, 80, 512),
    (4, 2048, 512, 8, 4, 64, 1024),
])
def test_block_bf16(p, S, hidden, Hq, Hkv, d, C):
    xin = gen.make_block_inputs("normal", 41, S, hidden, Hq, Hkv, d)
    got = run_block(xin, p, C, "bf16", Hq, Hkv, d)
    ref = oracle_block(xin, Hq, Hkv, d, "bf16")
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


@pytest.mark.parametrize("p", [1, 2])
def test_block_fp32(p):
    S, hidden, Hq, Hkv, d, C = 1024, 128, 4, 2, 64, 256
    xin = gen.make_block_inputs("normal", 42, S, hidden, Hq, Hkv, d)
    got = run_block(xin, p, C, "fp32", Hq, Hkv, d)
    ref = oracle_block(xin, Hq, Hkv, d, "fp32")
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["fp32"] for e in errs.values()), errs


def test_block_sparse():
    S, hidden, Hq, Hkv, d, C = 2048, 256, 4, 2, 64, 256
    keep = gen.sparsity_plan(S // C, 0.4, seed=9)
    xin = gen.make_block_inputs("normal", 43, S, hidden, Hq, Hkv, d)
    got = run_block(xin, 1, C, "bf16", Hq, Hkv, d, keep=keep)
    ref = oracle_block(xin, Hq, Hkv, d, "bf16", keep=keep, C=C)
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_block_errors():
    from paper_2408_16978_b200 import fpdt
    S, hidden, Hq, Hkv, d, C = 512, 128, 2, 2, 64, 256
    x = torch.zeros(S, hidden, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(hidden, (Hq + 2 * Hkv) * d, dtype=torch.bfloat16, device="cuda")
    o = torch.empty(S, Hq, d, dtype=torch.bfloat16, device="cuda")
    dx, dw = torch.empty_like(x), torch.empty(tuple(w.shape), dtype=torch.float32, device="cuda")
    q = torch.zeros(S, Hq, d, dtype=torch.bfloat16, device="cuda")
    ctx = fpdt.FPDTContext()
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_block_fwd(ctx, x, w, o, None, S, hidden, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 0)
    assert e.value.code == fpdt.FPDT_ERR_UNSUPPORTED
    fpdt.fpdt_attn_fwd(ctx, q, q, q, o, None, S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_block_bwd(ctx, x, w, o, o, dx, dw, S, hidden, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    assert e.value.code == fpdt.FPDT_ERR_STATE
    fpdt.fpdt_block_fwd(ctx, x, w, o, None, S, hidden, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    dq = torch.empty_like(q)
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_attn_bwd(ctx, o, o, dq, dq, dq, S, Hq, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
    assert e.value.code == fpdt.FPDT_ERR_STATE
    torch.cuda.synchronize()
    ctx.close()


@pytest.mark.parametrize("p,dtype", [(1, "bf16"), (2, "bf16"), (1, "fp32"), (2, "fp32")])
def test_block_with_output_projection(p, dtype):
    """y = attention(x W_qkv) W_o and the backward from dL/dy: y, dx, dW_qkv, dW_o against the oracle."""
    S, hidden, Hq, Hkv, d, C = 1024, 256, 4, 2, 64, 256
    xin = gen.make_block_inputs("normal", 44, S, hidden, Hq, Hkv, d)
    op = gen.make_output_proj_inputs(44, S, hidden, Hq, d)
    got = run_block(xin, p, C, dtype, Hq, Hkv, d, oproj=op)
    r = dtype == "bf16"
    o, lse = block.block_forward(xin["x"], xin["w"], Hq, Hkv, d, bf16_intermediates=r)
    y = block.output_forward(o, op["wo"], bf16_intermediates=r)
    do, dwo = block.output_backward(o, op["wo"], op["dy"], bf16_intermediates=r)
    dx, dw = block.block_backward(xin["x"], xin["w"], do, Hq, Hkv, d, bf16_intermediates=r)
    ref = {"o": o, "lse": lse, "y": y, "dx": dx, "dw": dw, "dwo": dwo}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL[dtype] for e in errs.values()), errs


def test_block_ragged_gemm_shapes():
    """Projection GEMM tiles that do not divide the problem: hidden = 200 (K and, for the output projection, N not a
    multiple of the 64 / 256 tile), Hq + 2 Hkv = 4 heads of d = 80 (N = 320), 256-row chunks."""
    S, hidden, Hq, Hkv, d, C = 1024, 200, 2, 1, 80, 256
    xin = gen.make_block_inputs("normal", 45, S, hidden, Hq, Hkv, d)
    op = gen.make_output_proj_inputs(45, S, hidden, Hq, d)
    got = run_block(xin, 1, C, "bf16", Hq, Hkv, d, oproj=op)
    o, lse = block.block_forward(xin["x"], xin["w"], Hq, Hkv, d, bf16_intermediates=True)
    y = block.output_forward(o, op["wo"], bf16_intermediates=True)
    do, dwo = block.output_backward(o, op["wo"], op["dy"], bf16_intermediates=True)
    dx, dw = block.block_backward(xin["x"], xin["w"], do, Hq, Hkv, d, bf16_intermediates=True)
    ref = {"o": o, "lse": lse, "y": y, "dx": dx, "dw": dw, "dwo": dwo}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_block_stress_world1():
    """The fused-projection block at p = 1 with u = 8 chunks under scheduler stress (random sleeps before every copy,
    GEMM and attention launch): the per-chunk projection of chunk m+2 writes the receive buffer chunk m's pairs read,
    so a missing event edge there shows up as wrong numbers."""
    from test_gpu_stress import stressed
    S, hidden, Hq, Hkv, d, C = 2048, 256, 4, 2, 64, 256
    xin = gen.make_block_inputs("normal", 46, S, hidden, Hq, Hkv, d)
    op = gen.make_output_proj_inputs(46, S, hidden, Hq, d)
    base = run_block(xin, 1, C, "bf16", Hq, Hkv, d, oproj=op)
    with stressed(seed=6):
        got = run_block(xin, 1, C, "bf16", Hq, Hkv, d, oproj=op)
    for n in ("o", "lse", "y"):
        assert np.array_equal(got[n], base[n]), n
    for n in ("dx", "dw", "dwo"):
        assert rel_err(got[n], base[n]) < 1e-2, n


@pytest.mark.parametrize("p", [1, 2])
def test_block_hidden_offload(p):
    """The forward offloads the hidden-state chunks and the backward, called with x = None, prefetches them for the
    projection backward: same O, dx, dW as with x on the device; the host link carries the x bytes."""
    S, hidden, Hq, Hkv, d, C = 2048, 256, 4, 2, 64, 512
    xin = gen.make_block_inputs("normal", 47, S, hidden, Hq, Hkv, d)
    st_a, st_b = {}, {}
    a = run_block(xin, p, C, "bf16", Hq, Hkv, d, stats=st_a)
    b = run_block(xin, p, C, "bf16", Hq, Hkv, d, hidden_offload=True, stats=st_b)
    for n in ("o", "lse"):
        assert np.array_equal(a[n], b[n]), n
    for n in ("dx", "dw"):
        assert rel_err(b[n], a[n]) < 1e-2, n
    ref = oracle_block(xin, Hq, Hkv, d, "bf16")
    errs = {n: rel_err(b[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    xbytes = (S // p) * hidden * 2
    for r in range(p):
        assert st_b[r]["bytes_d2h"] - st_a[r]["bytes_d2h"] == xbytes
        assert st_b[r]["bytes_h2d"] - st_a[r]["bytes_h2d"] == xbytes


@pytest.mark.parametrize("oproj", [False, True])
def test_block_one_rank_nccl(oproj):
    """The fused-projection block through a one-rank NCCL communicator: the forward GEMM's epilogue scatters into the
    all-to-all send layout and ncclAlltoAll delivers it; equal to the direct world-size-1 block (O, lse bitwise) and to
    the oracle."""
    S, hidden, Hq, Hkv, d, C = 2048, 320, 4, 4, 80, 512
    xin = gen.make_block_inputs("normal", 43, S, hidden, Hq, Hkv, d)
    op = gen.make_output_proj_inputs(45, S, hidden, Hq, d) if oproj else None
    got = run_block(xin, 1, C, "bf16", Hq, Hkv, d, oproj=op, nccl1=True)
    ref = run_block(xin, 1, C, "bf16", Hq, Hkv, d, oproj=op)
    assert np.array_equal(got["o"], ref["o"]) and np.array_equal(got["lse"], ref["lse"])
    for n in ("dx", "y") if oproj else ("dx",):
        assert rel_err(got[n], ref[n]) < 1e-2, n
    if not oproj:
        exact = oracle_block(xin, Hq, Hkv, d, "bf16")
        errs = {n: rel_err(got[n], exact[n]) for n in exact}
        assert all(e <= TOL["bf16"] for e in errs.values()), errs
