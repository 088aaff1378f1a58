"""Conditioning of the "drift32" inputs for dQ (R28), on the CPU with the fp64 oracle.

dQ_i = sigma sum_j dS_ij k_j is a sum whose terms cancel (sum_j dS_ij = 0 for the exact gradient), so a common offset
of the keys (drift32: up to 32 in one dimension) multiplies every perturbation of dS.  Any attention that forms the
forward output from bf16-rounded probabilities (the tensor-core PV product) feeds the backward a D_i = <dO_i, O_i>
that is not exactly sum_j P_ij dP_ij for the backward's own P, so sum_j dS_ij != 0 at the bf16 level, and the offset
turns that into a dQ error.  This test evaluates exactly that arithmetic -- the oracle's definition with only the
forward's P rounded to bf16 in O and everything else in fp64 -- and pins that its dQ error on drift32 is already of
the order of the 1e-2 bar while O, dK, dV stay far below it, and that the milder "drift" (8/S) keeps dQ well below.
The GPU path is held to 3e-2 on drift32's dQ (tests/test_gpu_extreme.py)."""
import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from oracle import attention


def _bf16(x):
    return torch.tensor(x).to(torch.bfloat16).to(torch.float64).numpy()


def _bf16p_forward_grads(x, h, g):
    """dQ and O of one head with O formed from bf16-rounded probabilities (exact otherwise)."""
    q, k, v, do = (x[n][:, i].astype(np.float64) for n, i in (("q", h), ("k", g), ("v", g), ("do", h)))
    S, d = q.shape
    sc = 1.0 / np.sqrt(d)
    s = np.where(np.tril(np.ones((S, S), bool)), sc * q @ k.T, -np.inf)
    m = s.max(1, keepdims=True)
    pt = np.exp(s - m)
    l = pt.sum(1, keepdims=True)
    o = (_bf16(pt) @ v) / l          # the forward's PV product with bf16 P
    p = pt / l                       # the backward's recomputed P
    ds = p * (do @ v.T - (do * o).sum(1, keepdims=True))
    return sc * ds @ k, o


@pytest.mark.parametrize("dist,lo,hi", [("drift32", 4e-3, 3e-2), ("drift", 0.0, 5e-3)])
def test_drift_dq_conditioning(dist, lo, hi):
    S, Hq, Hkv, d = 2048, 2, 1, 64
    x = gen.make_inputs(dist, 31, S, Hq, Hkv, d)
    o_ref, lse = attention.attention_forward(x["q"], x["k"], x["v"])
    dq_ref = attention.attention_backward(x["q"], x["k"], x["v"], o_ref, lse, x["do"])[0]
    worst = {"dq": 0.0, "o": 0.0}
    for h in range(Hq):
        dq, o = _bf16p_forward_grads(x, h, 0)
        worst["dq"] = max(worst["dq"], np.abs(dq - dq_ref[:, h]).max() / np.abs(dq_ref[:, h]).max())
        worst["o"] = max(worst["o"], np.abs(o - o_ref[:, h]).max() / np.abs(o_ref[:, h]).max())
    assert lo <= worst["dq"] <= hi, worst
    assert worst["o"] < 5e-3, worst
