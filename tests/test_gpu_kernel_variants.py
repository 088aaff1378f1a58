"""Every backward pair kernel against the fp64 oracle, launched directly (fpdt_debug_pair in libfpdt_diag.so) on the
causal diagonal pair of one chunk, so that each kernel is checked whether or not the library's dispatch picks it:
  2  attn_bwd_pipe_kernel   fp16 dQ product, d = 64 / 80 (the library's choice at 64 / 80); multicast CTA pairs sharing
                            the Q / dO loads when the key tiles pair up, single CTAs otherwise
  3  attn_bwd_2cta_kernel   CTA pair (tcgen05 cta_group::2), fp16 dQ product, d = 64 / 80 (diagnostics library only)
  4  attn_bwd_q64_kernel    64-row query tiles, d = 64 / 80 / 128 (the library's choice at 128); CTA pairs as 2
The forward statistics the backward consumes (log2-domain lse, D = rowsum(dO o O)) come from the oracle, so each
kernel's dQ, dK, dV are compared on their own (normwise max relative error <= 1e-2, bf16 I/O)."""
import ctypes

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, rel_err
from oracle import attention

pytestmark = pytest.mark.gpu


def _run(which, x, d, Hq, Hkv):
    from paper_2408_16978_b200 import fpdt
    lib = fpdt.diag()
    S = x["q"].shape[0]
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"])
    Dst = (x["do"].astype(np.float64) * o).sum(-1)                    # [S, Hq]
    bf = torch.bfloat16
    q, k, v, do = (torch.tensor(x[n]).to(bf).cuda().contiguous() for n in ("q", "k", "v", "do"))
    lse2 = torch.tensor((lse * np.log2(np.e)).T.copy(), dtype=torch.float32).cuda().contiguous()   # [Hq, S]
    dst = torch.tensor(Dst.T.copy(), dtype=torch.float32).cuda().contiguous()
    dq = torch.zeros(Hq, S, d, dtype=torch.float32, device="cuda")
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    rc = lib.fpdt_debug_pair(which, d, 1, P(q), P(k), P(v), P(do), P(lse2), P(dst), P(dq), P(dk), P(dv), S, Hq, Hkv,
                             None, 0, None)
    assert rc == 0, rc
    torch.cuda.synchronize()
    return {"dq": dq.permute(1, 0, 2).cpu().numpy(), "dk": dk.float().cpu().numpy(), "dv": dv.float().cpu().numpy()}, \
        (o, lse)


CASES = [(2, 64), (2, 80), (3, 64), (3, 80), (4, 64), (4, 80), (4, 128)]  # S = 1024: 8 key tiles, 4 CTA pairs


@pytest.mark.parametrize("which,d", CASES)
@pytest.mark.parametrize("dist,Hq,Hkv", [("normal", 2, 2), ("drift", 4, 2), ("extreme", 4, 1)])
def test_backward_kernel(which, d, dist, Hq, Hkv):
    S = 1024  # 8 key tiles (4 CTA pairs), 8 query tiles
    x = gen.make_inputs(dist, 71, S, Hq, Hkv, d)
    got, (o, lse) = _run(which, x, d, Hq, Hkv)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"])
    errs = {"dq": rel_err(got["dq"], dq), "dk": rel_err(got["dk"], dk), "dv": rel_err(got["dv"], dv)}
    assert all(np.isfinite(got[n]).all() for n in got)
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


@pytest.mark.parametrize("which,d", [(2, 80), (2, 64), (4, 128)])
@pytest.mark.parametrize("S", [1152, 1280])
def test_backward_kernel_cluster_parity(which, d, S):
    """The pipe (d = 64 / 80) and q64 (d = 128) kernels run in multicast CTA pairs when the key range has an even
    number of 128-row tiles (S = 1280: 10 tiles, 5 pairs, the second CTA of each diagonal pair starting on fully
    masked query tiles) and as single CTAs otherwise (S = 1152: 9 tiles); both against the oracle, GQA group 2."""
    x = gen.make_inputs("drift", 73, S, 4, 2, d)
    got, (o, lse) = _run(which, x, d, 4, 2)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"])
    errs = {"dq": rel_err(got["dq"], dq), "dk": rel_err(got["dk"], dk), "dv": rel_err(got["dv"], dv)}
    assert all(np.isfinite(got[n]).all() for n in got)
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
