"""FPDT-structured chunked attention over simulated ranks, step by step in the paper's order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Forward (fig:pipele_case0 and fig:pipele_case2), for every chunk
slot m = 0..u-1, all ranks in lockstep:
  1. slice T_m = rows [m c, (m+1) c) of every rank's local q, k, v;
  2. Alltoall: scatter heads, gather sequence -> q_m, k_m, v_m of shape
     [C, H/p, d] on every rank;
  3. attention of q_m with the resident k_m, v_m (diagonal block, causal) —
     for m = 0 this is already the final output;
  4. fetch k_i, v_i for i < m "chunk by chunk from the host memory"
     and update the output with the online-attention policy (
     recurrence = reading R2: running max m, denominator l, unnormalised o);
     at most one fetched set is checked out at any time;
  5. offload q_m, k_m, v_m to the host store;
  6. Alltoall back of the chunk output to its owner ranks.

Backward (fig:bw_db): the outer loop runs over key/value chunks j,
the inner loop over query chunks i >= j ("q_i never attends to k_j if i<j").
dk_j, dv_j accumulate across the inner loop and are final after outer
iteration j; dq_i accumulates across outer iterations in the host store
(reading R8) and is final after the inner iteration i = j.  D = rowsum(dO o O)
is computed in the sequence layout and moved with dO (reading R9).  The final
dq_j, dk_j, dv_j go back to their owner ranks by the reverse Alltoall.
"""
from __future__ import annotations

import numpy as np

from . import layout
from .attention import default_scale
from .store import ChunkStore


class OnlineState:
    """Running row max m, denominator l and unnormalised output o (reading R2)."""

    def __init__(self, n_rows: int, n_heads: int, head_dim: int):
        self.m = np.full((n_rows, n_heads), -np.inf)
        self.l = np.zeros((n_rows, n_heads))
        self.o = np.zeros((n_rows, n_heads, head_dim))

    def update(self, scores: np.ndarray, v: np.ndarray, G: int) -> None:
        """scores [h, rows, cols] (already scaled and masked with -inf); v [cols, hkv, d]."""
        for hh in range(scores.shape[0]):
            s = scores[hh]
            m_new = np.maximum(self.m[:, hh], s.max(axis=1))
            alpha = np.exp(self.m[:, hh] - m_new)          # 0 when m was -inf
            p = np.exp(s - m_new[:, None])
            self.l[:, hh] = alpha * self.l[:, hh] + p.sum(axis=1)
            self.o[:, hh] = alpha[:, None] * self.o[:, hh] + p @ v[:, hh // G]
            self.m[:, hh] = m_new

    def finalize(self):
        o = self.o / self.l[:, :, None]
        lse = self.m + np.log(self.l)
        return o, lse


def _block_scores(q: np.ndarray, k: np.ndarray, scale: float, G: int, diagonal: bool) -> np.ndarray:
    """[h, rows, cols] scores of a chunk pair; `diagonal` applies the within-chunk causal mask."""
    h = q.shape[1]
    s = np.stack([scale * (q[:, hh] @ k[:, hh // G].T) for hh in range(h)])
    if diagonal:
        n = s.shape[1]
        s = np.where((np.arange(n)[None, :] > np.arange(n)[:, None])[None], -np.inf, s)
    return s


def fpdt_forward(q_loc, k_loc, v_loc, chunk_size: int, scale: float | None = None,
                 host_capacity: int | None = None):
    """Per-rank local q [s_local, Hq, d], k/v [s_local, Hkv, d] (rank-ordinal order).

    Returns (o_loc, lse_loc, saved): per-rank outputs in the sequence layout and the
    saved state (host stores + head-layout lse) for `fpdt_backward`.
    """
    p = len(q_loc)
    s_local, Hq, d = q_loc[0].shape
    Hkv = k_loc[0].shape[1]
    c = chunk_size // p
    u = s_local // c
    G = Hq // Hkv
    scale = default_scale(d) if scale is None else scale
    stores = [ChunkStore(host_capacity) for _ in range(p)]
    lse_h = [[None] * u for _ in range(p)]
    o_loc = [np.zeros((s_local, Hq, d)) for _ in range(p)]
    lse_loc = [np.zeros((s_local, Hq)) for _ in range(p)]
    for m in range(u):
        rows = slice(m * c, (m + 1) * c)
        qh = layout.alltoall_seq2head([np.asarray(x[rows], np.float64) for x in q_loc])
        kh = layout.alltoall_seq2head([np.asarray(x[rows], np.float64) for x in k_loc])
        vh = layout.alltoall_seq2head([np.asarray(x[rows], np.float64) for x in v_loc])
        out_o, out_lse = [], []
        for rho in range(p):
            st = OnlineState(chunk_size, Hq // p, d)
            st.update(_block_scores(qh[rho], kh[rho], scale, G, diagonal=True), vh[rho], G)
            for i in range(m):
                kv_i = stores[rho].fetch(("kv", i))
                st.update(_block_scores(qh[rho], kv_i[0], scale, G, diagonal=False), kv_i[1], G)
                stores[rho].release(("kv", i))
            stores[rho].offload(("q", m), qh[rho])
            stores[rho].offload(("kv", m), np.stack([kh[rho], vh[rho]]))
            o_m, lse_m = st.finalize()
            lse_h[rho][m] = lse_m
            out_o.append(o_m)
            out_lse.append(lse_m[:, :, None])
        for r, (o_r, l_r) in enumerate(zip(layout.alltoall_head2seq(out_o), layout.alltoall_head2seq(out_lse))):
            o_loc[r][rows] = o_r
            lse_loc[r][rows] = l_r[:, :, 0]
    saved = {"stores": stores, "lse": lse_h, "p": p, "u": u, "c": c, "G": G, "scale": scale,
             "chunk_size": chunk_size}
    return o_loc, lse_loc, saved


def fpdt_backward(saved, o_loc, do_loc):
    """Nested-loop backward. Returns per-rank (dq_loc, dk_loc, dv_loc) in sequence layout."""
    if saved is None:
        raise RuntimeError("backward without saved forward state")
    p, u, c, G, scale = (saved[k] for k in ("p", "u", "c", "G", "scale"))
    stores, lse_h = saved["stores"], saved["lse"]
    s_local, Hq, d = o_loc[0].shape
    Hkv = Hq // G
    C = c * p
    dq_loc = [np.zeros((s_local, Hq, d)) for _ in range(p)]
    dk_loc = [np.zeros((s_local, Hkv, d)) for _ in range(p)]
    dv_loc = [np.zeros((s_local, Hkv, d)) for _ in range(p)]
    # B1: D = rowsum(dO o O) in the sequence layout (reading R9)
    D_loc = [np.einsum("shd,shd->sh", np.asarray(do, np.float64), np.asarray(o, np.float64))
             for do, o in zip(do_loc, o_loc)]
    # B2: per chunk, Alltoall dO (+D) to the head layout and offload dO_i
    D_h = [[None] * u for _ in range(p)]
    for m in range(u):
        rows = slice(m * c, (m + 1) * c)
        doh = layout.alltoall_seq2head([np.asarray(x[rows], np.float64) for x in do_loc])
        Dh = layout.alltoall_seq2head([x[rows][:, :, None] for x in D_loc])
        for rho in range(p):
            stores[rho].offload(("do", m), doh[rho])
            D_h[rho][m] = Dh[rho][:, :, 0]
    epoch = {}
    for j in range(u):                                   # outer loop: key / value chunk
        finals = []
        for rho in range(p):
            kv = stores[rho].fetch(("kv", j))
            k_j, v_j = kv[0], kv[1]
            dk_j = np.zeros((C, Hkv // p, d))
            dv_j = np.zeros((C, Hkv // p, d))
            epoch[(rho, j)] = j
            dq_final = None
            for i in range(j, u):                        # inner loop: query chunk i >= j
                q_i = stores[rho].fetch(("q", i))
                do_i = stores[rho].fetch(("do", i))
                dq_i = np.zeros((C, Hq // p, d)) if j == 0 else stores[rho].fetch(("dq", i))
                lse_i, D_i = lse_h[rho][i], D_h[rho][i]
                s = _block_scores(q_i, k_j, scale, G, diagonal=(i == j))
                for hh in range(Hq // p):
                    g = hh // G
                    P = np.exp(s[hh] - lse_i[:, hh][:, None])
                    dP = do_i[:, hh] @ v_j[:, g].T
                    dS = P * (dP - D_i[:, hh][:, None])
                    dq_i[:, hh] += scale * (dS @ k_j[:, g])
                    dk_j[:, g] += scale * (dS.T @ q_i[:, hh])
                    dv_j[:, g] += P.T @ do_i[:, hh]
                assert epoch[(rho, j)] == j              # dk_j / dv_j written only in outer iteration j
                if i == j:                               # last contribution: dq_j is final
                    dq_final = dq_i
                    if j > 0:
                        stores[rho].release(("dq", i))
                        stores[rho].free(("dq", i))
                elif j == 0:
                    stores[rho].offload(("dq", i), dq_i)
                else:
                    stores[rho].update(("dq", i), dq_i)
                    stores[rho].release(("dq", i))
                stores[rho].release(("q", i))
                stores[rho].release(("do", i))
            stores[rho].release(("kv", j))
            finals.append((dq_final, dk_j, dv_j))
        rows = slice(j * c, (j + 1) * c)            # reverse Alltoall of the final dq_j, dk_j, dv_j
        for dst, idx in ((dq_loc, 0), (dk_loc, 1), (dv_loc, 2)):
            for r, part in enumerate(layout.alltoall_head2seq([f[idx] for f in finals])):
                dst[r][rows] = part
    return dq_loc, dk_loc, dv_loc
