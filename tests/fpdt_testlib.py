"""Shared helpers for the GPU parity tests: run the CUDA path through the C-ABI binding, compare with the
oracle by the normwise max relative error of SURVEY §8(c) c.4."""
from __future__ import annotations

import numpy as np
import torch

import fpdt_inputs as gen
from oracle import attention

TOL = {"bf16": 1e-2, "fp32": 1e-4}   # north_star: 1e-2 for bf16 I/O with fp32 accumulation, 1e-4 fp32 mode


def rel_err(x, ref) -> float:
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-30))


def run_cuda(x: dict, chunk: int, dtype: str, offload: int, ctx=None, want_grad: bool = True, host_io: bool = False):
    """x: numpy q, k, v, do (bf16-representable fp32 values), sequence layout, world_size 1.
    host_io: every tensor in pinned host memory, through fpdt_attn_fwd_host / fpdt_attn_bwd_host."""
    from paper_2408_16978_b200 import fpdt
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    place = (lambda t: t.pin_memory()) if host_io else (lambda t: t.cuda())
    q, k, v, do = (place(torch.tensor(x[n]).to(tdt).contiguous()) for n in ("q", "k", "v", "do"))
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    own = ctx is None
    if own:
        ctx = fpdt.FPDTContext()
    empty = (lambda t: torch.empty_like(t).pin_memory()) if host_io else torch.empty_like
    o = empty(q)
    lse = empty(torch.empty(S, Hq, dtype=torch.float32, device=q.device))
    code = fpdt.dtype_code(tdt)
    fwd, bwd = (fpdt.fpdt_attn_fwd_host, fpdt.fpdt_attn_bwd_host) if host_io else (fpdt.fpdt_attn_fwd, fpdt.fpdt_attn_bwd)
    fwd(ctx, q, k, v, o, lse, S, Hq, Hkv, d, 1, chunk, 1, code, offload)
    out = {"o": o, "lse": lse}
    if want_grad:
        dq, dk, dv = empty(q), empty(k), empty(v)
        bwd(ctx, o, do, dq, dk, dv, S, Hq, Hkv, d, 1, chunk, 1, code, offload)
        out.update(dq=dq, dk=dk, dv=dv)
    torch.cuda.synchronize()
    res = {n: t.float().cpu().numpy() for n, t in out.items()}
    res["stats"] = ctx.stats()
    if own:
        ctx.close()
    return res


def oracle_full(x: dict):
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"])
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"])
    return {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}


def inputs(dist, seed, S, Hq, Hkv, d):
    return gen.make_inputs(dist, seed, S, Hq, Hkv, d)


def expected_bwd_bytes(order, u, C, Hq, Hkv, d, eb, keep=None, rkv=0, rq=0):
    """(H2D, D2H) bytes of the backward chunk loop, world size 1, excluding the dO offload of the preamble."""
    kv, qc = C * 2 * Hkv * d * eb, C * Hq * d * eb
    dqc, dkvc = C * Hq * d * 4, C * 2 * Hkv * d * 4
    kept = lambda i, j: i == j or keep is None or bool(keep[i][j])
    kres = lambda j: j < rkv
    qres = lambda i: i >= u - rq
    h2d = d2h = 0
    if order == 0:  # KV-outer (the paper's order); else Q-outer
        started = set()
        for j in range(u):
            h2d += 0 if kres(j) else kv
            for i in range(j, u):
                if not kept(i, j):
                    continue
                if not qres(i):
                    h2d += 2 * qc + (dqc if i in started else 0)
                    d2h += dqc if i != j else 0
                started.add(i)
    else:
        last = {j: max(i for i in range(j, u) if kept(i, j)) for j in range(u)}
        started = set()
        for i in range(u):
            h2d += 0 if qres(i) else 2 * qc
            for j in range(i + 1):
                if not kept(i, j):
                    continue
                if not kres(j):
                    h2d += kv + (dkvc if j in started else 0)
                    d2h += dkvc if i != last[j] else 0
                started.add(j)
    return h2d, d2h
