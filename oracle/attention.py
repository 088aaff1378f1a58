"""Plain definition of causal softmax attention and its gradient, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition (PAPER.md P:L112 for softmax(QK^T)V, P:L218 for
the causal mask, P:L171 for the backward input set q, k, v, o, dO; scale
sigma = 1/sqrt(d) is reading R1 in DESIGN.md because the paper never states it):

    s_ij   = sigma <q_i^h, k_j^g>                  j <= i (causal, diagonal included)
    lse_i  = log sum_{j<=i} exp(s_ij)
    O_i^h  = sum_{j<=i} exp(s_ij - lse_i) v_j^g
    D_i    = <dO_i^h, O_i^h>
    P_ij   = exp(s_ij - lse_i);   dP_ij = <dO_i^h, v_j^g>;   dS_ij = P_ij (dP_ij - D_i)
    dQ_i^h = sigma sum_j dS_ij k_j^g
    dK_j^g = sigma sum_{h in g} sum_i dS_ij q_i^h
    dV_j^g = sum_{h in g} sum_i P_ij dO_i^h

q-head h reads KV head g = h // G with G = Hq/Hkv (GQA; reading R12).

Block-sparse variant (§5.6: "only part of the tokens in key and value will be fetched from the
host memory, while the query will always be the entire sequence"; SPEC S:L102-103, S:L157 for the plan): with a
chunk size C and a plan keep[m][i] over (query chunk m, key chunk i), i <= m, key j is visible to query i iff
j <= i and keep[i // C][j // C]; diagonal blocks are always kept (every row attends to itself).
Shapes: q, o, dO [S, Hq, d]; k, v [S, Hkv, d]; lse, D [S, Hq].
The score matrix is materialised per head (brute force), with row-max
subtraction for a stable softmax; a library matmul serves as each product.
"""
from __future__ import annotations

import numpy as np


def default_scale(head_dim: int) -> float:
    return 1.0 / np.sqrt(head_dim)


def _scores(q_h: np.ndarray, k_g: np.ndarray, scale: float, causal: bool, keep=None, chunk: int = 0) -> np.ndarray:
    s = scale * (q_h @ k_g.T)
    if causal:
        n_q, n_k = s.shape
        # causal on global positions: row i attends j <= i (square case, S_q == S_k)
        mask = np.arange(n_k)[None, :] > np.arange(n_q)[:, None]
        if keep is not None:
            keep = np.asarray(keep, dtype=bool)
            blocks = keep[np.arange(n_q)[:, None] // chunk, np.arange(n_k)[None, :] // chunk]
            mask = mask | ~blocks
        s = np.where(mask, -np.inf, s)
    return s


def attention_forward(q, k, v, scale: float | None = None, causal: bool = True, keep=None, chunk: int = 0):
    """O, lse of the plain definition (block-sparse if keep [u,u] and chunk are given). fp64 (o [S,Hq,d], lse [S,Hq])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    scale = default_scale(d) if scale is None else scale
    o = np.empty((S, Hq, d))
    lse = np.empty((S, Hq))
    for h in range(Hq):
        g = h // G
        s = _scores(q[:, h], k[:, g], scale, causal, keep, chunk)
        m = s.max(axis=1, keepdims=True)
        e = np.exp(s - m)
        l = e.sum(axis=1, keepdims=True)
        o[:, h] = (e / l) @ v[:, g]
        lse[:, h] = (m + np.log(l))[:, 0]
    return o, lse


def attention_backward(q, k, v, o, lse, do, scale: float | None = None, causal: bool = True, keep=None,
                       chunk: int = 0):
    """dQ, dK, dV of L = sum(dO * O) by the definition above (fp64; block-sparse with keep / chunk)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    scale = default_scale(d) if scale is None else scale
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    D = np.einsum("shd,shd->sh", do, o)
    for h in range(Hq):
        g = h // G
        s = _scores(q[:, h], k[:, g], scale, causal, keep, chunk)
        P = np.exp(s - lse[:, h][:, None])          # exp(-inf) = 0 on masked entries
        dP = do[:, h] @ v[:, g].T
        dS = P * (dP - D[:, h][:, None])
        dq[:, h] = scale * (dS @ k[:, g])
        dk[:, g] += scale * (dS.T @ q[:, h])
        dv[:, g] += P.T @ do[:, h]
    return dq, dk, dv


def attention_probs(q, k, scale: float | None = None, causal: bool = True, head: int = 0, G: int = 1):
    """The softmax matrix P of one q-head (for invariant tests: rows sum to 1)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    scale = default_scale(q.shape[-1]) if scale is None else scale
    s = _scores(q[:, head], k[:, head // G], scale, causal)
    m = s.max(axis=1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=1, keepdims=True)
