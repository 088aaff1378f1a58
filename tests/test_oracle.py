"""Pins of the fp64 oracle against things other than itself (task rule ③).

Each test names what fixes the expected value: a library routine (torch SDPA /
autograd in fp64), a closed form, finite differences, a textbook special case,
the paper's own layout example, or an exact identity.
"""
import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from oracle import attention, closed_forms, fpdt, layout, sampled
from oracle.store import ChunkStore, StoreError


def _inputs(dist, S, Hq, Hkv, d, seed=0):
    x = gen.make_inputs(dist, seed, S, Hq, Hkv, d)
    return [x[n].astype(np.float64) for n in ("q", "k", "v", "do")]


def _torch_ref(q, k, v, do, causal=True):
    """Library routine: torch SDPA + autograd in fp64 (GQA by repeating KV heads)."""
    G = q.shape[1] // k.shape[1]
    tq = torch.tensor(q).permute(1, 0, 2).requires_grad_()
    tk = torch.tensor(k).permute(1, 0, 2).requires_grad_()
    tv = torch.tensor(v).permute(1, 0, 2).requires_grad_()
    o = torch.nn.functional.scaled_dot_product_attention(
        tq, tk.repeat_interleave(G, 0), tv.repeat_interleave(G, 0), is_causal=causal)
    o.backward(torch.tensor(do).permute(1, 0, 2))
    f = lambda t: t.detach().permute(1, 0, 2).numpy()
    return f(o), f(tq.grad), f(tk.grad), f(tv.grad)


# ---------------------------------------------------------------- generator
def test_generator_deterministic_bf16_and_moments():
    a = gen.generate("q", "normal", 3, np.arange(2048), 4, 64, 2048)
    b = gen.generate("q", "normal", 3, np.arange(2048), 4, 64, 2048)
    assert np.array_equal(a, b)
    assert np.array_equal(gen.bf16_round(a), a)              # bf16-representable
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1.1547) < 0.01   # Irwin-Hall(4) scaled
    c = gen.generate("q", "normal", 4, np.arange(2048), 4, 64, 2048)
    assert not np.array_equal(a, c)


def test_generator_rank_shards_are_global_rows():
    S, C, p = 256, 64, 4
    full = gen.generate("k", "normal", 0, np.arange(S), 2, 8, S)
    for r in range(p):
        toks = gen.global_tokens_of_rank(r, p, S // p, C)
        assert np.array_equal(gen.generate("k", "normal", 0, toks, 2, 8, S), full[toks])
    shards = layout.shard(full, p, S // C)
    for r in range(p):
        assert np.array_equal(shards[r], full[gen.global_tokens_of_rank(r, p, S // p, C)])


def test_bf16_round_nearest_even():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1.0 + 2 ** -9], np.float32)
    np.testing.assert_array_equal(gen.bf16_round(x), np.array([1.0, 1.0, 1.0 + 4 * 2 ** -8, -2.5, 1.0], np.float32))


# ---------------------------------------------------------------- plain definition
@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (4, 2), (8, 1)])
def test_definition_matches_torch_sdpa_fp64(Hq, Hkv):
    q, k, v, do = _inputs("normal", 96, Hq, Hkv, 16)
    o, lse = attention.attention_forward(q, k, v)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do)
    to, tdq, tdk, tdv = _torch_ref(q, k, v, do)
    for a, b in ((o, to), (dq, tdq), (dk, tdk), (dv, tdv)):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


def test_noncausal_definition_matches_torch():
    q, k, v, do = _inputs("normal", 40, 2, 2, 8)
    o, lse = attention.attention_forward(q, k, v, causal=False)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do, causal=False)
    to, tdq, tdk, tdv = _torch_ref(q, k, v, do, causal=False)
    for a, b in ((o, to), (dq, tdq), (dk, tdk), (dv, tdv)):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


def test_lse_matches_logsumexp_library():
    from scipy.special import logsumexp
    q, k, v, _ = _inputs("peaky", 50, 2, 2, 8)
    _, lse = attention.attention_forward(q, k, v)
    s = (q[:, 1] @ k[:, 1].T) / np.sqrt(8)
    ref = np.array([logsumexp(s[i, : i + 1]) for i in range(50)])
    np.testing.assert_allclose(lse[:, 1], ref, rtol=0, atol=1e-12)


def test_single_token_output_is_v():
    q, k, v, _ = _inputs("normal", 1, 2, 2, 8)
    o, lse = attention.attention_forward(q, k, v)
    np.testing.assert_array_equal(o, v)
    np.testing.assert_allclose(lse, (q * k).sum(-1) / np.sqrt(8), atol=1e-15)


def test_rows_sum_to_one_and_causal_zeros():
    q, k, _, _ = _inputs("normal", 64, 2, 2, 8)
    P = attention.attention_probs(q, k, head=1)
    np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-12)
    assert np.all(np.triu(P, 1) == 0.0)


def test_identical_keys_prefix_mean():                   # SPEC S:L115, closed form
    S, H, d = 128, 2, 8
    x = gen.make_inputs("same", 1, S, H, H, d)
    q, k, v = (x[n].astype(np.float64) for n in ("q", "k", "v"))
    assert np.array_equal(k[0], k[77])
    o, lse = attention.attention_forward(q, k, v)
    prefix = np.stack([v[: t + 1].mean(0) for t in range(S)])
    np.testing.assert_allclose(o, prefix, atol=1e-13)
    np.testing.assert_allclose(lse, (q * k[0][None]).sum(-1) / np.sqrt(d) + np.log(np.arange(1, S + 1))[:, None],
                               atol=1e-12)
    o2, lse2 = closed_forms.identical_keys_forward(q, k[0], v)
    np.testing.assert_allclose(o2, prefix, atol=1e-13)
    np.testing.assert_allclose(lse2, lse, atol=1e-12)
    dq, _, _ = attention.attention_backward(q, k, v, o, lse, x["do"].astype(np.float64))
    np.testing.assert_allclose(dq, 0.0, atol=1e-12)       # identical keys: dQ = 0


def test_finite_difference_gradient():                   # SPEC S:L142 (FD, fp64, step 1e-5)
    S, H, d, C = 32, 2, 4, 8
    q, k, v, do = _inputs("normal", S, H, H, d, seed=2)
    o_l, lse_l, saved = fpdt.fpdt_forward([q], [k], [v], C)
    dq, dk, dv = fpdt.fpdt_backward(saved, o_l, [do])
    loss = lambda q_, k_, v_: float((attention.attention_forward(q_, k_, v_)[0] * do).sum())
    rng = np.random.default_rng(0)
    eps = 1e-5
    for name, g, x in (("q", dq[0], q), ("k", dk[0], k), ("v", dv[0], v)):
        for _ in range(12):
            idx = tuple(rng.integers(0, n) for n in x.shape)
            xp, xm = x.copy(), x.copy()
            xp[idx] += eps
            xm[idx] -= eps
            args_p = {"q": (xp, k, v), "k": (q, xp, v), "v": (q, k, xp)}[name]
            args_m = {"q": (xm, k, v), "k": (q, xm, v), "v": (q, k, xm)}[name]
            fd = (loss(*args_p) - loss(*args_m)) / (2 * eps)
            assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, g[idx])


def test_zero_upstream_gives_zero_gradients():
    q, k, v, do = _inputs("normal", 32, 2, 1, 8)
    o, lse, saved = fpdt.fpdt_forward([q], [k], [v], 8)
    dq, dk, dv = fpdt.fpdt_backward(saved, o, [np.zeros_like(do)])
    for g in (dq[0], dk[0], dv[0]):
        assert np.all(g == 0.0)


# ---------------------------------------------------------------- FPDT structure == definition
@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("u", [1, 2, 4, 8])
@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (8, 4)])
def test_fpdt_structured_equals_definition(p, u, Hq, Hkv):   # chunk-count & world-size invariance
    S, d = 128, 8
    if Hkv % p:
        pytest.skip("GQA under Ulysses needs Hkv % p == 0")
    q, k, v, do = _inputs("drift", S, Hq, Hkv, d, seed=u + p)
    o, lse = attention.attention_forward(q, k, v)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do)
    C = S // u
    shards = [layout.shard(x, p, u) for x in (q, k, v, do)]
    o_l, lse_l, saved = fpdt.fpdt_forward(shards[0], shards[1], shards[2], C)
    np.testing.assert_allclose(layout.unshard(o_l, u), o, rtol=0, atol=1e-10)
    np.testing.assert_allclose(layout.unshard(lse_l, u), lse, rtol=0, atol=1e-10)
    for st in saved["stores"]:
        assert st.highwater <= 1                           # "only one set of chunks"
    dq_l, dk_l, dv_l = fpdt.fpdt_backward(saved, o_l, shards[3])
    for a, b in ((dq_l, dq), (dk_l, dk), (dv_l, dv)):
        np.testing.assert_allclose(layout.unshard(a, u), b, rtol=0, atol=1e-9)


def test_fpdt_extreme_logits_merge():
    S, H, d = 64, 2, 8
    q, k, v, do = _inputs("normal", S, H, H, d, seed=7)
    q = q * 30.0                                            # logits ~ +-100s
    o, lse = attention.attention_forward(q, k, v)
    o_l, lse_l, _ = fpdt.fpdt_forward([q], [k], [v], 8)
    np.testing.assert_allclose(o_l[0], o, atol=1e-10)
    np.testing.assert_allclose(lse_l[0], lse, rtol=1e-14, atol=1e-10)


def test_fpdt_backward_requires_forward():
    with pytest.raises(RuntimeError):
        fpdt.fpdt_backward(None, [np.zeros((8, 1, 4))], [np.zeros((8, 1, 4))])


def test_fpdt_host_capacity_error():
    q, k, v, _ = _inputs("normal", 64, 2, 2, 8)
    need = 64 * 2 * 8 * 8 * 3                               # q, k, v chunks of all slots, fp64
    fpdt.fpdt_forward([q], [k], [v], 16, host_capacity=need)
    with pytest.raises(StoreError):
        fpdt.fpdt_forward([q], [k], [v], 16, host_capacity=need - 1)


# ---------------------------------------------------------------- causality & metamorphic
def test_causality_bitwise():
    q, k, v, _ = _inputs("normal", 64, 2, 2, 8)
    o, lse, _ = fpdt.fpdt_forward([q], [k], [v], 16)
    k2, v2 = k.copy(), v.copy()
    k2[40:] += 3.0
    v2[40:] -= 1.0
    o2, lse2, _ = fpdt.fpdt_forward([q], [k2], [v2], 16)
    assert np.array_equal(o[0][:32], o2[0][:32]) and np.array_equal(lse[0][:32], lse2[0][:32])


def test_key_shift_invariance():
    q, k, v, do = _inputs("normal", 48, 2, 2, 8)
    c = np.linspace(-1, 1, 8)
    o, lse = attention.attention_forward(q, k, v)
    o2, lse2 = attention.attention_forward(q, k + c[None, None, :], v)
    np.testing.assert_allclose(o2, o, atol=1e-12)
    np.testing.assert_allclose(lse2 - lse, (q @ c) / np.sqrt(8), atol=1e-12)
    g1 = attention.attention_backward(q, k, v, o, lse, do)
    g2 = attention.attention_backward(q, k + c, v, o2, lse2, do)
    for a, b in zip(g1, g2):
        np.testing.assert_allclose(a, b, atol=1e-11)


def test_gradient_identities():
    q, k, v, do = _inputs("sink", 96, 4, 2, 8)
    o, lse = attention.attention_forward(q, k, v)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do)
    np.testing.assert_allclose(dk.sum(0), 0.0, atol=1e-12)      # sum_j dS_ij = 0
    np.testing.assert_allclose(dv.sum(0), do.reshape(96, 2, 2, 8).sum((0, 2)), atol=1e-12)  # rows of P sum to 1


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("Hq,Hkv", [(2, 2), (4, 1)])
def test_class_keys_closed_form_matches_definition(Hq, Hkv):
    S, d = 256, 8
    x = gen.make_inputs("class", 5, S, Hq, Hkv, d)
    q, k, v, do = (x[n].astype(np.float64) for n in ("q", "k", "v", "do"))
    cls = gen.class_of(np.arange(S), S)
    kc = np.stack([k[np.argmax(cls == c)] for c in range(gen.N_CLASSES)])
    for c in range(gen.N_CLASSES):
        assert np.all(k[cls == c] == kc[c])
    G = Hq // Hkv
    o, lse = attention.attention_forward(q, k, v)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do)
    o2, lse2 = closed_forms.class_keys_forward(q, kc, cls, v, G=G)
    np.testing.assert_allclose(o2, o, atol=1e-12)
    np.testing.assert_allclose(lse2, lse, atol=1e-12)
    dq2, dk2, dv2 = closed_forms.class_keys_backward(q, kc, cls, v, do, G=G, block=48)
    for a, b in ((dq2, dq), (dk2, dk), (dv2, dv)):
        np.testing.assert_allclose(a, b, atol=1e-11)


# ---------------------------------------------------------------- sampled rows / tail columns
def test_sampled_rows_and_tail_columns_match_definition():
    S, Hq, Hkv, d = 160, 4, 2, 8
    q, k, v, do = _inputs("drift", S, Hq, Hkv, d)
    o, lse = attention.attention_forward(q, k, v)
    dq, dk, dv = attention.attention_backward(q, k, v, o, lse, do)
    rows = np.array([0, 1, 63, 64, 100, 159])
    sc = 1 / np.sqrt(d)
    dq_r, o_r, lse_r = sampled.rows_dq(q[rows, 3], do[rows, 3], rows, k[:, 1], v[:, 1], sc)
    np.testing.assert_allclose(o_r, o[rows, 3], atol=1e-13)
    np.testing.assert_allclose(lse_r, lse[rows, 3], atol=1e-13)
    np.testing.assert_allclose(dq_r, dq[rows, 3], atol=1e-12)
    t0 = S - 24
    dk_t, dv_t = sampled.tail_dkdv(q[t0:, 2:4].transpose(1, 0, 2), do[t0:, 2:4].transpose(1, 0, 2), t0,
                                   k[:, 1], v[:, 1], sc)
    np.testing.assert_allclose(dk_t, dk[t0:, 1], atol=1e-12)
    np.testing.assert_allclose(dv_t, dv[t0:, 1], atol=1e-12)


# ---------------------------------------------------------------- layout (paper example)
def test_paper_layout_example():
    p = u = 4
    assert [layout.naive_subchunk(r, 1, u) for r in range(p)] == [1, 5, 9, 13]
    assert [layout.global_subchunk(r, 1, p) for r in range(p)] == [4, 5, 6, 7]


@pytest.mark.parametrize("p,u", [(1, 1), (2, 4), (4, 2), (4, 4), (8, 2)])
def test_shard_alltoall_roundtrip_and_contiguity(p, u):
    S, H, d = 8 * p * u, 2 * p, 3
    x = np.arange(S * H * d, dtype=np.float64).reshape(S, H, d)    # sentinel = flat index
    loc = layout.shard(x, p, u)
    assert np.array_equal(layout.unshard(loc, u), x)
    c = S // (p * u)
    for m in range(u):
        recv = layout.alltoall_seq2head([l[m * c:(m + 1) * c] for l in loc])
        for rho in range(p):                                # contiguous global range, own heads
            assert np.array_equal(recv[rho], x[m * p * c:(m + 1) * p * c, rho * (H // p):(rho + 1) * (H // p)])
        back = layout.alltoall_head2seq(recv)
        for r in range(p):
            assert np.array_equal(back[r], loc[r][m * c:(m + 1) * c])


def test_pack_index_sentinel_oracle():
    p, c, H, d = 2, 4, 2, 1                                  # SPEC S:L202 exhaustive p=2 case
    chunks = [np.arange(c * H * d).reshape(c, H, d) + 1000 * r for r in range(p)]
    idx = layout.pack_index(p, c, H, d)
    recv = layout.alltoall_seq2head(chunks)
    for rho in range(p):
        # block from rank r in rho's receive buffer == rank r's packed segment for destination rho
        seg = [chunks[r].reshape(-1)[idx].reshape(p, c, H // p, d)[rho] for r in range(p)]
        assert np.array_equal(np.concatenate(seg, 0), recv[rho])
    assert len(set(idx.tolist())) == c * H * d              # a permutation; equal bytes per peer


def test_store_semantics():
    st = ChunkStore(capacity_bytes=64)
    st.offload("a", np.zeros(4))                            # 32 B
    st.offload("b", np.zeros(4))                            # exactly capacity
    with pytest.raises(StoreError):
        st.offload("c", np.zeros(1))
    with pytest.raises(StoreError):
        st.fetch("zz")
    assert np.array_equal(st.fetch("a"), np.zeros(4))
    st.release("a")
    st.free("a")
    with pytest.raises(StoreError):
        st.free("a")


def test_generator_head_subset_matches_full():
    """The oracle regenerates single heads at full size: a head subset must equal those heads of the full tensor."""
    toks = np.array([0, 5, 1023, 4096, 70000])
    for dist in ("normal", "drift", "class"):
        full = gen.generate("k", dist, 4, toks, 8, 16, 100000)
        sub = gen.generate("k", dist, 4, toks, 8, 16, 100000, heads=[1, 6])
        assert np.array_equal(full[:, [1, 6]], sub)


def test_sparsity_plan_properties():
    for u, rho in ((8, 0.0), (8, 0.25), (8, 0.5), (4, 0.9)):
        keep = gen.sparsity_plan(u, rho, seed=3)
        assert keep.shape == (u, u) and keep.dtype == bool
        assert np.all(np.diag(keep)) and not np.any(np.triu(keep, 1))
        n_valid = u * (u + 1) // 2
        assert n_valid - keep.sum() == min(int(np.floor(rho * n_valid)), u * (u - 1) // 2)
        assert np.array_equal(keep, gen.sparsity_plan(u, rho, seed=3))


def test_block_sparse_definition_pins():
    """Block-sparse oracle pins (§5.6): all-kept == dense; diagonal-only == independent per-chunk causal
    attention; a random plan == torch SDPA (fp64) with the explicit boolean block mask; and the backward of that
    plan == autograd through the same SDPA."""
    S, Hq, Hkv, d, C = 96, 4, 2, 16, 24
    u = S // C
    x = gen.make_inputs("normal", 5, S, Hq, Hkv, d)
    dense = attention.attention_forward(x["q"], x["k"], x["v"])
    allk = attention.attention_forward(x["q"], x["k"], x["v"], keep=np.tril(np.ones((u, u), bool)), chunk=C)
    np.testing.assert_allclose(allk[0], dense[0], rtol=0, atol=1e-13)
    diag = attention.attention_forward(x["q"], x["k"], x["v"], keep=np.eye(u, dtype=bool), chunk=C)
    for m in range(u):
        sl = slice(m * C, (m + 1) * C)
        o_m, lse_m = attention.attention_forward(x["q"][sl], x["k"][sl], x["v"][sl])
        np.testing.assert_allclose(diag[0][sl], o_m, rtol=0, atol=1e-13)
        np.testing.assert_allclose(diag[1][sl], lse_m, rtol=0, atol=1e-13)
    keep = gen.sparsity_plan(u, 0.4, seed=1)
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
    do = x["do"]
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, do, keep=keep, chunk=C)
    t = {n: torch.tensor(x[n], dtype=torch.float64, requires_grad=(n != "do")) for n in ("q", "k", "v", "do")}
    G = Hq // Hkv
    visible = (torch.arange(S)[None, :] <= torch.arange(S)[:, None]) & torch.tensor(
        keep[np.arange(S)[:, None] // C, np.arange(S)[None, :] // C])
    qh = t["q"].permute(1, 0, 2)
    kh = t["k"].repeat_interleave(G, dim=1).permute(1, 0, 2)
    vh = t["v"].repeat_interleave(G, dim=1).permute(1, 0, 2)
    ref = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, attn_mask=visible).permute(1, 0, 2)
    np.testing.assert_allclose(o, ref.detach().numpy(), rtol=0, atol=1e-12)
    (ref * t["do"]).sum().backward()
    np.testing.assert_allclose(dq, t["q"].grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(dk, t["k"].grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(dv, t["v"].grad.numpy(), rtol=0, atol=1e-11)
