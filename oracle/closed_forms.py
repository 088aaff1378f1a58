"""Closed forms of causal attention for structured keys — exact at any sequence length.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

These are consequences of the plain definition (oracle/attention.py) when keys
take only a few distinct values; they let parity be checked on every output
element at full BASELINE sizes in O(S K d) (forward, dV) or O(S B d) (dK),
where the brute force would need O(S^2 d).  SURVEY §8(c) c.3.

Identical keys (k_j = k for all j):
    O_t = mean(v_0..v_t),  lse_t = sigma <q_t, k> + ln(t+1),  dQ = 0.

Class keys (k_j = k_{c(j)}, classes c = 0..K-1), per q-head h with KV head g:
    s_tc   = sigma <q_t, k_c>,  n_c(t) = #{j<=t: c(j)=c},  V_c(t) = sum_{j<=t, c(j)=c} v_j
    lse_t  = M_t + ln sum_c n_c(t) e^{s_tc - M_t},   M_t = max_{c: n_c(t)>0} s_tc
    O_t    = sum_c e^{s_tc - lse_t} V_c(t)
    P_tc   = e^{s_tc - lse_t}  (the probability of ONE key of class c in row t)
    D_t    = <dO_t, O_t>
    dQ_t   = sigma sum_c P_tc (<dO_t, V_c(t)> - D_t n_c(t)) k_c
    dV_j   = sum_{h in g} sum_{t>=j} P_{t,c(j)} dO_t
    dK_j   = sigma sum_{h in g} sum_{t>=j} P_{t,c(j)} (<dO_t, v_j> - D_t) q_t
The dK sum is evaluated block-wise: a carried suffix matrix
M_c = sum_{t >= block end} P_tc q_t dO_t^T (d x d) plus the in-block lower
triangle, which is the same sum regrouped (associativity of +).
"""
from __future__ import annotations

import numpy as np

from .attention import default_scale


def identical_keys_forward(q, k_row, v, scale: float | None = None, G: int = 1):
    """q [S,Hq,d]; k_row [Hkv,d] (the one key); v [S,Hkv,d]. Returns (o, lse)."""
    q = np.asarray(q, np.float64)
    v = np.asarray(v, np.float64)
    k_row = np.asarray(k_row, np.float64)
    S, Hq, d = q.shape
    scale = default_scale(d) if scale is None else scale
    counts = np.arange(1, S + 1, dtype=np.float64)
    prefix_mean = np.cumsum(v, axis=0) / counts[:, None, None]
    heads = np.arange(Hq) // G
    o = prefix_mean[:, heads]
    lse = scale * np.einsum("shd,hd->sh", q, k_row[heads]) + np.log(counts)[:, None]
    return o, lse


def class_keys_forward(q, k_classes, cls, v, scale: float | None = None, G: int = 1):
    """q [S,Hq,d]; k_classes [K,Hkv,d]; cls [S] int class of each key; v [S,Hkv,d]."""
    q = np.asarray(q, np.float64)
    v = np.asarray(v, np.float64)
    kc = np.asarray(k_classes, np.float64)
    S, Hq, d = q.shape
    K = kc.shape[0]
    scale = default_scale(d) if scale is None else scale
    onehot = (np.asarray(cls)[:, None] == np.arange(K)[None, :]).astype(np.float64)   # [S,K]
    n = np.cumsum(onehot, axis=0)                                                    # n_c(t)
    o = np.empty_like(q)
    lse = np.empty((S, Hq))
    for h in range(Hq):
        g = h // G
        Vc = np.cumsum(onehot[:, :, None] * v[:, g][:, None, :], axis=0)             # [S,K,d]
        s = scale * q[:, h] @ kc[:, g].T                                             # [S,K]
        s_valid = np.where(n > 0, s, -np.inf)
        M = s_valid.max(axis=1)
        lse[:, h] = M + np.log((n * np.exp(s_valid - M[:, None])).sum(axis=1))
        w = np.exp(s_valid - lse[:, h][:, None])                                     # P_tc
        o[:, h] = np.einsum("sk,skd->sd", w, Vc)
    return o, lse


def class_keys_backward(q, k_classes, cls, v, do, scale: float | None = None, G: int = 1,
                        block: int = 512):
    """dQ, dK, dV by the class-keys closed form (see module docstring)."""
    q = np.asarray(q, np.float64)
    v = np.asarray(v, np.float64)
    do = np.asarray(do, np.float64)
    kc = np.asarray(k_classes, np.float64)
    cls = np.asarray(cls)
    S, Hq, d = q.shape
    Hkv = kc.shape[1]
    K = kc.shape[0]
    scale = default_scale(d) if scale is None else scale
    o, lse = class_keys_forward(q, kc, cls, v, scale, G)
    D = np.einsum("shd,shd->sh", do, o)
    onehot = (cls[:, None] == np.arange(K)[None, :]).astype(np.float64)
    n = np.cumsum(onehot, axis=0)
    dq = np.zeros_like(q)
    dk = np.zeros((S, Hkv, d))
    dv = np.zeros((S, Hkv, d))
    for h in range(Hq):
        g = h // G
        Vc = np.cumsum(onehot[:, :, None] * v[:, g][:, None, :], axis=0)
        s = scale * q[:, h] @ kc[:, g].T
        P = np.where(n > 0, np.exp(s - lse[:, h][:, None]), 0.0)                     # [S,K]
        inner = np.einsum("sd,skd->sk", do[:, h], Vc) - D[:, h][:, None] * n
        dq[:, h] = scale * (P * inner) @ kc[:, g]
        # dV_j = sum_{t>=j} P_{t,c(j)} dO_t : reverse cumulative sums per class
        suffix_dv = np.cumsum((P[:, :, None] * do[:, h][:, None, :])[::-1], axis=0)[::-1]   # [S,K,d]
        dv[:, g] += suffix_dv[np.arange(S), cls]
        # dK_j = sigma sum_{t>=j} P_{t,c(j)} (<dO_t, v_j> - D_t) q_t
        suffix_dq = np.cumsum(((P * D[:, h][:, None])[:, :, None] * q[:, h][:, None, :])[::-1], axis=0)[::-1]
        part2 = suffix_dq[np.arange(S), cls]                                         # sum P D q
        part1 = np.zeros((S, d))
        carry = np.zeros((K, d, d))                                                  # sum_{t>=end} P_tc q_t dO_t^T
        for end in range(S, 0, -block):
            start = max(0, end - block)
            qb, dob, vb, Pb, cb = q[start:end, h], do[start:end, h], v[start:end, g], P[start:end], cls[start:end]
            # carried part: (M_c v_j) for each j in block
            part1[start:end] = np.einsum("jde,je->jd", carry[cb], vb)
            # in-block part: sum_{t in block, t >= j} P_{t,c(j)} q_t <dO_t, v_j>
            L = dob @ vb.T                                                           # [t, j] = <dO_t, v_j>
            W = Pb[:, cb] * L                                                        # [t, j] = P_{t,c(j)} <dO_t,v_j>
            W = np.where(np.arange(end - start)[:, None] >= np.arange(end - start)[None, :], W, 0.0)
            part1[start:end] += W.T @ qb
            carry += np.einsum("tc,td,te->cde", Pb, qb, dob)
        dk[:, g] += scale * (part1 - part2)
    return dq, dk, dv
