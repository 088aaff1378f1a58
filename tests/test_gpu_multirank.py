"""The p > 1 path (all-to-all pack/unpack, per-chunk exchange, head-sharded attention, reverse exchange) on ONE
GPU: p ranks of an in-process group (fpdt_group_create), one host thread and one stream per rank.

Checks (SURVEY §8(c) c.3 "invariances", c.5): world-size invariance against the p = 1 run of the same GLOBAL
inputs — bitwise for O, lse, dK, dV (per-head arithmetic is identical and there are no atomics on them),
within tolerance for dQ (its fp32 reduce-add order varies) — and oracle parity at p > 1."""
import threading

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, oracle_full, rel_err

pytestmark = pytest.mark.gpu


def run_group(x: dict, p: int, C: int, dtype: str, offload: int, keep=None, residency=None, bwd_order=None,
              stats=None, fetch=None, debug_checks=False, host_io=False) -> dict:
    """Shard the global inputs x by the rank-ordinal contract, run fwd+bwd on p local ranks, unshard."""
    from paper_2408_16978_b200 import fpdt
    S, Hq, d = x["q"].shape
    Hkv = x["k"].shape[1]
    s_local = S // p
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = fpdt.dtype_code(tdt)
    group = fpdt.LocalGroup(p) if p > 1 else None
    rows = [gen.global_tokens_of_rank(r, p, s_local, C) for r in range(p)]
    out = {n: np.zeros(x[m].shape, np.float32) for n, m in (("o", "q"), ("dq", "q"), ("dk", "k"), ("dv", "v"))}
    out["lse"] = np.zeros((S, Hq), np.float32)
    errors = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                place = (lambda t: t.pin_memory()) if host_io else (lambda t: t.cuda())
                q, k, v, do = (place(torch.tensor(x[n][rows[r]]).to(tdt).contiguous()) for n in ("q", "k", "v", "do"))
                empty = (lambda t: torch.empty_like(t).pin_memory()) if host_io else torch.empty_like
                o = empty(q)
                lse = empty(torch.empty(s_local, Hq, dtype=torch.float32, device=q.device))
                dq, dk, dv = empty(q), empty(k), empty(v)
            stream.synchronize()
            ctx = fpdt.FPDTContext(p, r, group=group) if p > 1 else fpdt.FPDTContext()
            if keep is not None:
                ctx.set_sparsity(keep)
            if residency is not None:
                ctx.set_residency(*residency)
            if bwd_order is not None:
                ctx.set_bwd_order(bwd_order)
            if fetch is not None:
                ctx.set_fetch_strategy(fetch)
            if debug_checks:
                ctx.set_debug_checks(True)
            fwd, bwd = ((fpdt.fpdt_attn_fwd_host, fpdt.fpdt_attn_bwd_host) if host_io
                        else (fpdt.fpdt_attn_fwd, fpdt.fpdt_attn_bwd))
            fwd(ctx, q, k, v, o, lse, s_local, Hq, Hkv, d, 1, C, p, code, offload, 0.0, stream)
            bwd(ctx, o, do, dq, dk, dv, s_local, Hq, Hkv, d, 1, C, p, code, offload, 0.0, stream)
            stream.synchronize()
            for n, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
                out[n][rows[r]] = t.float().cpu().numpy()
            if stats is not None:
                stats[r] = ctx.stats()
            ctx.close()
        except Exception as e:  # surfaced in the main thread
            errors.append((r, e))

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(p)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "a rank hung"
    if group is not None:
        group.close()
    assert not errors, errors
    return out


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("offload", [1, 0])
def test_world_size_invariance_bf16(p, offload):
    S, Hq, Hkv, d, C = 2048, 8, 4, 80, 512      # u = 4 chunks, GQA G = 2, head_dim of GPT-2.7B
    x = gen.make_inputs("drift", 7, S, Hq, Hkv, d)
    ref = run_group(x, 1, C, "bf16", offload)
    got = run_group(x, p, C, "bf16", offload)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], ref[n]), (n, rel_err(got[n], ref[n]))
    assert rel_err(got["dq"], ref["dq"]) < 1e-3


@pytest.mark.parametrize("p,S,Hq,Hkv,d,C", [
    (2, 2048, 4, 4, 64, 512),      # MHA, u = 4
    (4, 2048, 8, 4, 128, 1024),    # GQA G = 2, u = 2, c = 256 rows per rank
    (2, 1024, 8, 2, 128, 256),     # GQA G = 4 (Llama-3 8B ratio), smallest chunk
])
def test_oracle_parity_multirank_bf16(p, S, Hq, Hkv, d, C):
    x = gen.make_inputs("normal", 8, S, Hq, Hkv, d)
    ref = oracle_full(x)
    got = run_group(x, p, C, "bf16", 1)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_oracle_parity_multirank_fp32():
    S, Hq, Hkv, d, C = 1024, 4, 2, 64, 512
    x = gen.make_inputs("sink", 9, S, Hq, Hkv, d)
    ref = oracle_full(x)
    got = run_group(x, 2, C, "fp32", 1)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["fp32"] for e in errs.values()), errs


@pytest.mark.parametrize("p,Hq,Hkv", [
    (4, 32, 8),    # Llama-3 8B ratio (BASELINE configs[2]: 32 q / 8 kv heads, d = 128) at p = 4
    (8, 64, 8),    # 70B ratio (configs[4]: 64 q / 8 kv heads) at p = 8: one kv head per rank
])
def test_gqa_configs_sampled_rows(p, Hq, Hkv):
    """BASELINE configs[2] / [4] head shapes and world sizes at a reduced sequence (S = 16K, chunk 4K): sampled rows
    of O, lse, dQ against the oracle's single-row definition, and the dK/dV identities on every kv head."""
    from oracle import sampled
    S, d, C = 16384, 128, 4096
    x = gen.make_inputs("drift", 11, S, Hq, Hkv, d)
    got = run_group(x, p, C, "bf16", 1)
    rows = np.array(sorted(set([0, 1, 255, 256, C - 1, C, S - 1, 2 * C + 77, 3 * C + 4000, 9999])))
    G = Hq // Hkv
    for h in (0, Hq - 1):
        g = h // G
        dq, o, lse = sampled.rows_dq(x["q"][rows, h], x["do"][rows, h], rows, x["k"][:, g].astype(np.float64),
                                     x["v"][:, g].astype(np.float64), sampled.default_scale(d))
        errs = {"o": rel_err(got["o"][rows, h], o), "lse": rel_err(got["lse"][rows, h], lse),
                "dq": rel_err(got["dq"][rows, h], dq)}
        assert all(e <= TOL["bf16"] for e in errs.values()), (h, errs)
    dk_sum, dk_abs = got["dk"].sum(0), np.abs(got["dk"]).sum(0)
    assert np.max(np.abs(dk_sum) / dk_abs) <= TOL["bf16"]
    dv_sum, dv_abs = got["dv"].sum(0), np.abs(got["dv"]).sum(0)
    do_sum = x["do"].reshape(S, Hkv, G, d).sum(axis=(0, 2))
    assert np.max(np.abs(dv_sum - do_sum) / dv_abs) <= TOL["bf16"]


def test_block_sparse_multirank():
    """Block-sparse plan (§5.6) over global chunk indices at p = 2: equals the block-masked oracle."""
    from oracle import attention
    S, Hq, Hkv, d, C = 2048, 4, 2, 80, 256
    keep = gen.sparsity_plan(S // C, 0.4, seed=2)
    x = gen.make_inputs("normal", 13, S, Hq, Hkv, d)
    got = run_group(x, 2, C, "bf16", 1, keep=keep)
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"], keep=keep, chunk=C)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"], keep=keep, chunk=C)
    ref = {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


@pytest.mark.parametrize("residency", [(1, 1), (2, 3), (4, 4)])
def test_residency_multirank(residency):
    """HBM residency budget (include/fpdt.h fpdt_set_residency) at p = 2: resident head-layout chunks and (O, dO)
    chunks stay on the device; O, lse, dK, dV bitwise equal to the fully offloaded run, dQ within its reduce order,
    and the oracle."""
    S, Hq, Hkv, d, C = 2048, 4, 2, 80, 512   # u = 4
    x = gen.make_inputs("normal", 14, S, Hq, Hkv, d)
    base = run_group(x, 2, C, "bf16", 1)
    got = run_group(x, 2, C, "bf16", 1, residency=residency)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), (n, residency)
    assert rel_err(got["dq"], base["dq"]) < 1e-3
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
