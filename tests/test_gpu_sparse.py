"""Block-sparse FPDT attention (§5.6: only part of the key/value chunks are fetched from host memory and
computed; the query always covers the whole sequence) through the C-ABI, against the block-masked oracle definition
(oracle/attention.py, keep / chunk), at p = 1 and through the local multi-rank group."""
import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, rel_err
from oracle import attention

pytestmark = pytest.mark.gpu


def _oracle(x, keep, C):
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"], keep=keep, chunk=C)
    return {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}


def _run(x, C, keep, dtype="bf16"):
    from paper_2408_16978_b200 import fpdt
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, k, v, do = (torch.tensor(x[n]).to(tdt).cuda().contiguous() for n in ("q", "k", "v", "do"))
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    ctx = fpdt.FPDTContext()
    ctx.set_sparsity(keep)
    o = torch.empty_like(q)
    lse = torch.empty(S, Hq, dtype=torch.float32, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    code = fpdt.dtype_code(tdt)
    fpdt.fpdt_attn_fwd(ctx, q, k, v, o, lse, S, Hq, Hkv, d, 1, C, 1, code, 1)
    fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, Hq, Hkv, d, 1, C, 1, code, 1)
    torch.cuda.synchronize()
    st = ctx.stats()
    ctx.close()
    return {n: t.float().cpu().numpy() for n, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv))}, st


@pytest.mark.parametrize("rho", [0.25, 0.5])
@pytest.mark.parametrize("dtype,d", [("bf16", 80), ("bf16", 128), ("fp32", 64)])
def test_block_sparse_parity(rho, dtype, d):
    S, Hq, Hkv, C = 2048, 4, 2, 256
    u = S // C
    keep = gen.sparsity_plan(u, rho, seed=7)
    x = gen.make_inputs("normal", 12, S, Hq, Hkv, d)
    got, st = _run(x, C, keep, dtype)
    ref = _oracle(x, keep, C)
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL[dtype] for e in errs.values()), errs
    # dropped key chunks are never fetched: forward fetches = kept off-diagonal blocks
    kv_chunk = C * 2 * Hkv * d * (2 if dtype == "bf16" else 4)
    n_off = int(np.tril(keep, -1).sum())
    assert st["bytes_h2d"] >= n_off * kv_chunk


def test_sparse_plan_errors():
    from paper_2408_16978_b200 import fpdt
    S, H, d, C = 1024, 2, 64, 256
    t = lambda: torch.zeros(S, H, d, dtype=torch.bfloat16, device="cuda")
    q, k, v, o = t(), t(), t(), t()
    ctx = fpdt.FPDTContext()
    ctx.set_sparsity(np.tril(np.ones((3, 3), bool)))            # wrong chunk count
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, H, d, 1, C, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_ARG
    bad = np.tril(np.ones((4, 4), bool))
    bad[2, 2] = False                                            # dropped diagonal
    ctx.set_sparsity(bad)
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, H, d, 1, C, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_ARG
    ctx.set_sparsity(gen.sparsity_plan(4, 0.3))
    with pytest.raises(fpdt.FpdtError) as e:                     # resident mode has no per-pair schedule
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, H, d, 1, C, 1, 0, 0)
    assert e.value.code == fpdt.FPDT_ERR_UNSUPPORTED
    ctx.set_sparsity(None)
    fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, H, d, 1, C, 1, 0, 1)
    ctx.close()
