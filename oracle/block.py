"""Attention block with the chunked QKV projection fused in front, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:L206: "For the first QKV projection, since tokens are processed elementwise, we directly slice the local
sequence tensor into u chunks ... T_i is projected to query q_i, key k_i, and value v_i.  Then, we perform the
Alltoall"; after dq_0, dk_0, dv_0 are final and all-to-all'd back, they "are used to compute the gradient of
the input hidden state dc_0".  The projection is token-wise, so chunking does not change it; the plain definition
over the whole sequence is the oracle:

    [q | k | v] = x W                        x [S, hidden], W [hidden, (Hq + 2 Hkv) d] (columns q heads, k, v)
    O, lse      = attention(q, k, v)         (oracle/attention.py, §8(c) c.1)
    dq, dk, dv  = attention backward for dO
    dqkv        = [dq | dk | dv]             [S, (Hq + 2 Hkv) d]
    dx          = dqkv W^T                   (the hidden-state gradient, "dc" in P:L365)
    dW          = x^T dqkv                   (summed over every token of the sequence shard)

(no bias: the paper states none).

bf16 mode (reading R27 in DESIGN.md; the paper states no precision, R15): in a bf16 block the projected q, k, v and
the attention gradients dq, dk, dv that enter the projection backward are bf16 tensors, as every activation of a
bf16 layer is.  `bf16_intermediates=True` rounds them (RNE, via fp32) at exactly those two points; every product
and sum stays fp64.

Pinned in tests/test_oracle_block.py by central finite differences of the
scalar loss L = <dO, O> in x and W, and by reduction to the attention oracle when W selects x's columns.
"""
from __future__ import annotations

import numpy as np

from . import attention


def _bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 (ties to even) through fp32, returned as fp64."""
    u = np.ascontiguousarray(np.asarray(x, np.float64).astype(np.float32)).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32).astype(np.float64)


def split_qkv(qkv: np.ndarray, n_q_heads: int, n_kv_heads: int, head_dim: int):
    S = qkv.shape[0]
    nq, nk = n_q_heads * head_dim, n_kv_heads * head_dim
    q = qkv[:, :nq].reshape(S, n_q_heads, head_dim)
    k = qkv[:, nq:nq + nk].reshape(S, n_kv_heads, head_dim)
    v = qkv[:, nq + nk:].reshape(S, n_kv_heads, head_dim)
    return q, k, v


def _project(x, w, bf16_intermediates: bool):
    qkv = np.asarray(x, np.float64) @ np.asarray(w, np.float64)
    return _bf16(qkv) if bf16_intermediates else qkv


def block_forward(x, w, n_q_heads: int, n_kv_heads: int, head_dim: int, scale: float | None = None,
                  bf16_intermediates: bool = False):
    """O [S, Hq, d], lse [S, Hq] of attention over the projected q, k, v (causal)."""
    q, k, v = split_qkv(_project(x, w, bf16_intermediates), n_q_heads, n_kv_heads, head_dim)
    return attention.attention_forward(q, k, v, scale)


def block_backward(x, w, do, n_q_heads: int, n_kv_heads: int, head_dim: int, scale: float | None = None,
                   bf16_intermediates: bool = False, keep=None, chunk: int = 0):
    """dx [S, hidden], dW [hidden, (Hq + 2 Hkv) d] for upstream dO of the attention output (and O, lse)."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    S = x.shape[0]
    q, k, v = split_qkv(_project(x, w, bf16_intermediates), n_q_heads, n_kv_heads, head_dim)
    o, lse = attention.attention_forward(q, k, v, scale, keep=keep, chunk=chunk)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, np.asarray(do, np.float64), scale, keep=keep,
                                              chunk=chunk)
    dqkv = np.concatenate([dq.reshape(S, -1), dk.reshape(S, -1), dv.reshape(S, -1)], axis=1)
    if bf16_intermediates:
        dqkv = _bf16(dqkv)
    return dqkv @ w.T, x.T @ dqkv


# Output projection after the attention (the other side of the path; the paper's block ends in
# the attention output's projection before the FFN): y = O W_o with O flattened per token to [S, Hq d]
# (head-major, head_dim fastest) and W_o [Hq d, hidden]; backward dO = dY W_o^T, dW_o = O^T dY.  bf16 mode (R27):
# O and dO are bf16 tensors.
def output_forward(o, w_o, bf16_intermediates: bool = False):
    of = np.asarray(o, np.float64).reshape(np.shape(o)[0], -1)
    if bf16_intermediates:
        of = _bf16(of)
    return of @ np.asarray(w_o, np.float64)


def output_backward(o, w_o, dy, bf16_intermediates: bool = False):
    """dO [S, Hq, d] (the upstream gradient of the attention output) and dW_o [Hq d, hidden]."""
    S = np.shape(o)[0]
    of = np.asarray(o, np.float64).reshape(S, -1)
    if bf16_intermediates:
        of = _bf16(of)
    dy = np.asarray(dy, np.float64)
    do = dy @ np.asarray(w_o, np.float64).T
    if bf16_intermediates:
        do = _bf16(do)
    return do.reshape(np.shape(o)), of.T @ dy
