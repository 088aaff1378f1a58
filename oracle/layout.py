"""Sequence layout algebra of FPDT over simulated ranks (index permutations only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Rank-ordinal shuffle (fig:seq_shuffle): with p
  ranks and u chunks per rank, the global sequence is cut into p*u sub-chunks
  T_0..T_{pu-1} of c = S/(p u) tokens; rank r holds T_{i p + r} in its local
  slot i.  Gathering slot i across ranks then yields the contiguous token
  range T_{ip}..T_{ip+p-1}, so the ordinary causal mask stays valid.
  The naive layout (rank r holds T_{r u + i}) would gather T_1, T_5, T_9, T_13
  for slot 1 at p=u=4.
* Ulysses all-to-all: per slot, every rank sends its
  [c, H, d] chunk split by head blocks; rank rho receives the head block
  [rho*H/p, (rho+1)*H/p) of every rank, concatenated in rank order ->
  [C = p c, H/p, d] ("the Alltoall is an index permutation").
  Head blocks are contiguous (reading R11).
"""
from __future__ import annotations

import numpy as np


def global_subchunk(rank: int, slot: int, world_size: int) -> int:
    """Global sub-chunk index held by (rank, slot) in the shuffled layout."""
    return slot * world_size + rank


def naive_subchunk(rank: int, slot: int, chunks_per_rank: int) -> int:
    """Global sub-chunk index held by (rank, slot) in the unshuffled layout."""
    return rank * chunks_per_rank + slot


def global_token(rank: int, local_t: int, chunk_size: int, world_size: int) -> int:
    c = chunk_size // world_size
    return global_subchunk(rank, local_t // c, world_size) * c + local_t % c


def shard(x: np.ndarray, world_size: int, n_chunks: int) -> list:
    """Global [S, H, d] -> per-rank local [S/p, H, d] in rank-ordinal order."""
    S = x.shape[0]
    c = S // (world_size * n_chunks)
    out = []
    for r in range(world_size):
        parts = [x[global_subchunk(r, i, world_size) * c:(global_subchunk(r, i, world_size) + 1) * c]
                 for i in range(n_chunks)]
        out.append(np.concatenate(parts, axis=0))
    return out


def unshard(locals_: list, n_chunks: int) -> np.ndarray:
    """Inverse of `shard`."""
    p = len(locals_)
    c = locals_[0].shape[0] // n_chunks
    S = c * p * n_chunks
    out = np.empty((S,) + locals_[0].shape[1:], dtype=locals_[0].dtype)
    for r in range(p):
        for i in range(n_chunks):
            g = global_subchunk(r, i, p)
            out[g * c:(g + 1) * c] = locals_[r][i * c:(i + 1) * c]
    return out


def alltoall_seq2head(send: list) -> list:
    """send[r]: rank r's [c, H, d] slot chunk -> recv[rho]: [p*c, H/p, d] (heads of rho, all ranks' rows)."""
    p = len(send)
    c, H = send[0].shape[0], send[0].shape[1]
    hp = H // p
    recv = []
    for rho in range(p):
        blocks = [send[r][:, rho * hp:(rho + 1) * hp] for r in range(p)]
        recv.append(np.concatenate(blocks, axis=0))
    assert all(b.shape[0] == c for b in blocks)
    return recv


def alltoall_head2seq(send: list) -> list:
    """Inverse of alltoall_seq2head: send[rho]: [p*c, H/p, d] -> recv[r]: [c, H, d]."""
    p = len(send)
    C, hp = send[0].shape[0], send[0].shape[1]
    c = C // p
    recv = []
    for r in range(p):
        recv.append(np.concatenate([send[rho][r * c:(r + 1) * c] for rho in range(p)], axis=1))
    return recv


def pack_index(world_size: int, c: int, H: int, d: int):
    """Sentinel index oracle of the pack step: for packed element (dst, t, hh, e) of a rank's send
    buffer [p][c][H/p][d], the source element (t, dst*H/p + hh, e) of its [c, H, d] slot chunk.
    Returns an int64 array of flat source offsets in packed order."""
    hp = H // world_size
    dst = np.arange(world_size).reshape(-1, 1, 1, 1)
    t = np.arange(c).reshape(1, -1, 1, 1)
    hh = np.arange(hp).reshape(1, 1, -1, 1)
    e = np.arange(d).reshape(1, 1, 1, -1)
    return ((t * H + dst * hp + hh) * d + e).reshape(-1)
