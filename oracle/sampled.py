"""Single rows and tail columns of the plain definition, for parity at full BASELINE sizes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Row i of O, lse and dQ depends only on q_i, dO_i and keys/values j <= i
(definition in oracle/attention.py), so it costs O(i d) per head.  Column j of
dK, dV needs every row i >= j (their lse_i and D_i), so columns are taken in
the last `tail` tokens of the sequence, where that set is small.
Inputs are regenerated per row/head from ``fpdt_inputs`` by the caller.
"""
from __future__ import annotations

import numpy as np

from .attention import default_scale


def rows_forward(q_rows, row_idx, k_g, v_g, scale: float):
    """q_rows [R,d] of one head at global positions row_idx; k_g, v_g [>= max+1, d] its KV head.

    Returns (o [R,d], lse [R]) of the plain definition (causal, diagonal included)."""
    q_rows = np.asarray(q_rows, np.float64)
    o = np.empty_like(q_rows)
    lse = np.empty(len(row_idx))
    for r, i in enumerate(row_idx):
        s = scale * (k_g[: i + 1] @ q_rows[r])
        m = s.max()
        e = np.exp(s - m)
        l = e.sum()
        o[r] = (e / l) @ v_g[: i + 1]
        lse[r] = m + np.log(l)
    return o, lse


def rows_dq(q_rows, do_rows, row_idx, k_g, v_g, scale: float):
    """dQ rows [R,d] (and o, lse) of one head by the definition; D_i from the oracle's own O_i."""
    o, lse = rows_forward(q_rows, row_idx, k_g, v_g, scale)
    do_rows = np.asarray(do_rows, np.float64)
    dq = np.empty_like(o)
    for r, i in enumerate(row_idx):
        s = scale * (k_g[: i + 1] @ q_rows[r])
        P = np.exp(s - lse[r])
        dP = v_g[: i + 1] @ do_rows[r]
        D = do_rows[r] @ o[r]
        dq[r] = scale * ((P * (dP - D)) @ k_g[: i + 1])
    return dq, o, lse


def tail_dkdv(q_tail, do_tail, tail_start: int, k_g, v_g, scale: float):
    """dK, dV of KV head g for columns j in [tail_start, S) (S = len(k_g)).

    q_tail / do_tail: [G, S - tail_start, d] — the q-heads of the group for rows >= tail_start.
    Uses rows_forward for every row i >= tail_start (their lse_i and D_i)."""
    S = k_g.shape[0]
    T = S - tail_start
    Gh, _, d = q_tail.shape
    dk = np.zeros((T, d))
    dv = np.zeros((T, d))
    rows = np.arange(tail_start, S)
    for h in range(Gh):
        o, lse = rows_forward(q_tail[h], rows, k_g, v_g, scale)
        D = np.einsum("rd,rd->r", np.asarray(do_tail[h], np.float64), o)
        kt, vt = k_g[tail_start:], v_g[tail_start:]
        s = scale * (np.asarray(q_tail[h], np.float64) @ kt.T)           # [rows i, cols j]
        s = np.where(np.arange(T)[None, :] > np.arange(T)[:, None], -np.inf, s)
        P = np.exp(s - lse[:, None])
        dP = np.asarray(do_tail[h], np.float64) @ vt.T
        dS = P * (dP - D[:, None])
        dk += scale * (dS.T @ np.asarray(q_tail[h], np.float64))
        dv += P.T @ np.asarray(do_tail[h], np.float64)
    return dk, dv


__all__ = ["rows_forward", "rows_dq", "tail_dkdv", "default_scale"]
