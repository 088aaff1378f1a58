"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no attention, no softmax, no
layout algebra beyond "which global token is this row").  It is the one piece
of code both sides may use (task rule ③): the oracle calls the numpy twin
below, the GPU tests/bench call the bitwise-identical device twin in
``gen_dev.cu`` (``libfpdt_gen.so``).

Generator (documented so any implementation can reproduce it, cf. SPEC S:L68
"a fixed, well-known ... counter-based ... generator, specified in docs"):

    mix32(x)     = lowbias32: x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16
    a            = mix32(seed*0x9E3779B9 + tensor*0x85EBCA6B + 0x632BE5AB)     (mod 2^32)
    idx          = (token*H + head)*D + dim                (64-bit, GLOBAL token index)
    h1           = mix32(mix32(a ^ hi32(idx)) ^ lo32(idx))
    h2           = mix32(h1 + 0x9E3779B9)
    n            = (h1&0xffff) + (h1>>16) + (h2&0xffff) + (h2>>16) - 131070   (Irwin-Hall of 4)
    x            = n * 2^-15                               (exact in fp32; std ~1.155)
    value        = bf16_rne(transform(x))                  (all inputs are bf16-representable)

Distributions (SURVEY §8(c) "Input distributions"; transforms are single
IEEE fp32 ops so the device twin matches bitwise):

    normal : x
    peaky  : q*4                                                    (sharp attention)
    drift  : q[...,0] += 2 ;  k[t,...,0] += t*(8/S)                 (running max rises every chunk: the ramp moves
             the logits of the last keys by ~2*8/sqrt(d) = 1.4 nats (d = 128) over the sequence)
    drift32: the same with k[t,...,0] += t*(32/S)                   (~5.7 nats; adversarial for dQ: the key offset
             -- up to 32 in one dimension, ~3x the norm of the rest of a key -- multiplies the rounding error of any
             bf16 attention's dQ, R28)
    sink   : q += 0.5 ;  k[0] = 2 (all dims)                         (attention sink on token 0)
    same   : k[t] = base(K, token 0)                                (identical keys: closed form)
    class  : k[t] = base(K, token c(t)), c(t) = mix32(t^0xC1A55) % 3 for t < S/2, % 4 for t >= S/2;
             class 3 is scaled by 4 (a large-norm class that appears only in later chunks, so the
             running max jumps at chunk boundaries)
    extreme: q*30                                                   (logits of +-100s of nats: the online rescale
             under large max jumps, and keys far enough below the row max that exp2 underflows)
"""
from __future__ import annotations

import numpy as np

Q, K, V, DO, X, W, WO, DY = 0, 1, 2, 3, 4, 5, 6, 7
TENSOR_IDS = {"q": Q, "k": K, "v": V, "do": DO, "x": X, "w": W, "wo": WO, "dy": DY}
DISTRIBUTIONS = ("normal", "peaky", "drift", "sink", "same", "class", "extreme", "drift32")
DIST_IDS = {name: i for i, name in enumerate(DISTRIBUTIONS)}
N_CLASSES = 4


def _mix32(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint32(16))
    x = x * np.uint32(0x7FEB352D)
    x = x ^ (x >> np.uint32(15))
    x = x * np.uint32(0x846CA68B)
    x = x ^ (x >> np.uint32(16))
    return x


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest-even bf16, returned as fp32 (finite inputs only)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    bias = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + bias) & np.uint32(0xFFFF0000)).view(np.float32)


def base_values(seed: int, tensor: int, tokens: np.ndarray, n_heads: int, head_dim: int,
                heads: np.ndarray | None = None) -> np.ndarray:
    """Raw Irwin-Hall values (fp32, before bf16 rounding) for rows `tokens` (global token ids).

    Returns shape [len(tokens), n_heads, head_dim], or [len(tokens), len(heads), head_dim] for a subset of the
    n_heads heads (the values are those of the full tensor: the counter uses n_heads).
    """
    with np.errstate(over="ignore"):
        tok = np.asarray(tokens, dtype=np.uint64).reshape(-1, 1, 1)
        hsel = np.arange(n_heads) if heads is None else np.asarray(heads)
        hd = hsel.astype(np.uint64).reshape(1, -1, 1)
        dd = np.arange(head_dim, dtype=np.uint64).reshape(1, 1, -1)
        idx = (tok * np.uint64(n_heads) + hd) * np.uint64(head_dim) + dd
        a = _mix32(np.uint32((seed * 0x9E3779B9 + tensor * 0x85EBCA6B + 0x632BE5AB) & 0xFFFFFFFF))
        hi = (idx >> np.uint64(32)).astype(np.uint32)
        lo = (idx & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        h1 = _mix32(_mix32(a ^ hi) ^ lo)
        h2 = _mix32(h1 + np.uint32(0x9E3779B9))
        n = ((h1 & np.uint32(0xFFFF)).astype(np.int64) + (h1 >> np.uint32(16)).astype(np.int64)
             + (h2 & np.uint32(0xFFFF)).astype(np.int64) + (h2 >> np.uint32(16)).astype(np.int64) - 131070)
    return (n.astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float32)


def class_of(tokens: np.ndarray, seq_len: int) -> np.ndarray:
    """Key class c(t) of the 'class' distribution."""
    with np.errstate(over="ignore"):
        t = np.asarray(tokens, dtype=np.uint64)
        h = _mix32((t & np.uint64(0xFFFFFFFF)).astype(np.uint32) ^ np.uint32(0xC1A55))
        m = np.where(t >= np.uint64(seq_len // 2), np.uint32(4), np.uint32(3))
        return (h % m).astype(np.int64)


def generate(name: str, dist: str, seed: int, tokens: np.ndarray, n_heads: int, head_dim: int,
             seq_len: int, heads: np.ndarray | None = None) -> np.ndarray:
    """Values (fp32 holding bf16-representable numbers) of tensor `name` for global `tokens`.

    `seq_len` is the GLOBAL sequence length S (used by drift/class).  Shape [T, n_heads, head_dim], or
    [T, len(heads), head_dim] for a subset `heads` of the tensor's n_heads heads.
    """
    tensor = TENSOR_IDS[name]
    tokens = np.asarray(tokens, dtype=np.int64)
    if dist not in DIST_IDS:
        raise ValueError(f"unknown distribution {dist!r}")
    if name == "k" and dist in ("same", "class"):
        cls = np.zeros_like(tokens) if dist == "same" else class_of(tokens, seq_len)
        x = base_values(seed, tensor, cls, n_heads, head_dim, heads)
        if dist == "class":
            x = np.where((cls == 3).reshape(-1, 1, 1), x * np.float32(4.0), x).astype(np.float32)
        return bf16_round(x)
    x = base_values(seed, tensor, tokens, n_heads, head_dim, heads)
    if dist == "peaky" and name == "q":
        x = x * np.float32(4.0)
    elif dist == "extreme" and name == "q":
        x = x * np.float32(30.0)
    elif dist in ("drift", "drift32"):
        if name == "q":
            x[..., 0] = x[..., 0] + np.float32(2.0)
        elif name == "k":
            step = np.float32((8.0 if dist == "drift" else 32.0) / seq_len)
            x[..., 0] = x[..., 0] + (tokens.astype(np.float32) * step).reshape(-1, 1)
    elif dist == "sink":
        if name == "q":
            x = x + np.float32(0.5)
        elif name == "k":
            x[tokens == 0] = np.float32(2.0)
    return bf16_round(x.astype(np.float32))


def global_tokens_of_rank(rank: int, world_size: int, s_local: int, chunk_size: int) -> np.ndarray:
    """Global token id of each of rank `rank`'s local rows (the rank-ordinal input contract).

    Rank r's local token t is global token ((t div c)*p + r)*c + (t mod c), c = chunk_size/p
    (fig:seq_shuffle).  Pure index bookkeeping: this is the
    *input contract*, shared so both sides generate the same shard, not part of the method.
    """
    c = chunk_size // world_size
    t = np.arange(s_local, dtype=np.int64)
    return ((t // c) * world_size + rank) * c + (t % c)


def make_inputs(dist: str, seed: int, seq_len: int, n_q_heads: int, n_kv_heads: int, head_dim: int,
                tokens: np.ndarray | None = None) -> dict:
    """q, k, v, do (fp32 arrays of bf16-representable values) for the given global tokens."""
    if tokens is None:
        tokens = np.arange(seq_len, dtype=np.int64)
    return {
        "q": generate("q", dist, seed, tokens, n_q_heads, head_dim, seq_len),
        "k": generate("k", dist, seed, tokens, n_kv_heads, head_dim, seq_len),
        "v": generate("v", dist, seed, tokens, n_kv_heads, head_dim, seq_len),
        "do": generate("do", dist, seed, tokens, n_q_heads, head_dim, seq_len),
    }


def sparsity_plan(n_chunks: int, rho: float, seed: int = 0) -> np.ndarray:
    """Block-sparsity plan keep[m][i] (bool, [u,u]) over (query chunk m, key chunk i) — an INPUT of the method
    (§5.6 "block sparse attention"): every causally valid block i <= m is kept
    except floor(rho * u(u+1)/2) off-diagonal blocks chosen by a seeded permutation; diagonal blocks are never
    dropped (capped at all off-diagonal blocks); blocks i > m are False (causally invisible)."""
    u = int(n_chunks)
    keep = np.tril(np.ones((u, u), dtype=bool))
    off = [(m, i) for m in range(u) for i in range(m)]
    n_drop = min(int(np.floor(rho * u * (u + 1) / 2)), len(off))
    if n_drop:
        rng = np.random.default_rng(np.uint64(seed) * np.uint64(0x9E3779B9) + np.uint64(u))
        for idx in rng.permutation(len(off))[:n_drop]:
            keep[off[idx]] = False
    return keep


def make_block_inputs(dist: str, seed: int, seq_len: int, hidden: int, n_q_heads: int, n_kv_heads: int,
                      head_dim: int, tokens: np.ndarray | None = None) -> dict:
    """Inputs of the attention block with the fused QKV projection: the hidden state
    x [T, hidden] (rows = global tokens), the projection weight w [hidden, (Hq + 2 Hkv) * head_dim] (columns: q heads,
    then k heads, then v heads, head_dim fastest) scaled by 2^-round(log2(sqrt(hidden))) (exact in bf16) so the
    projected q, k, v have about unit variance, and the upstream gradient do [T, Hq, head_dim] of the attention
    output.  `dist` shapes x only through the base generator (normal); the attention-level distributions apply to
    q, k, v, which are now computed."""
    if tokens is None:
        tokens = np.arange(seq_len, dtype=np.int64)
    n_cols = (n_q_heads + 2 * n_kv_heads) * head_dim
    x = generate("x", "normal", seed, tokens, 1, hidden, seq_len).reshape(len(tokens), hidden)
    w = generate("w", "normal", seed, np.arange(hidden), 1, n_cols, seq_len).reshape(hidden, n_cols)
    w = (w * np.float32(2.0 ** -round(np.log2(np.sqrt(hidden))))).astype(np.float32)
    do = generate("do", dist, seed, tokens, n_q_heads, head_dim, seq_len)
    return {"x": x, "w": w, "do": do}


def make_output_proj_inputs(seed: int, seq_len: int, hidden: int, n_q_heads: int, head_dim: int,
                            tokens: np.ndarray | None = None) -> dict:
    """Output projection weight wo [Hq * head_dim, hidden] (scaled by 2^-round(log2(sqrt(Hq * head_dim)))) and the
    upstream gradient dy [T, hidden] of the block output y = o wo (rows = global tokens)."""
    if tokens is None:
        tokens = np.arange(seq_len, dtype=np.int64)
    k = n_q_heads * head_dim
    wo = generate("wo", "normal", seed, np.arange(k), 1, hidden, seq_len).reshape(k, hidden)
    wo = (wo * np.float32(2.0 ** -round(np.log2(np.sqrt(k))))).astype(np.float32)
    dy = generate("dy", "normal", seed, tokens, 1, hidden, seq_len).reshape(len(tokens), hidden)
    return {"wo": wo, "dy": dy}
