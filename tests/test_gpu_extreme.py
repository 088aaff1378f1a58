"""The online-softmax edge cases on the GPU (SURVEY §8(c) c.3 "online merge": extreme logits; "the
output ... will be rescaled in the next chunk computation").

Two input distributions of fpdt_inputs:
  * drift32 — k[t, 0] += 32 t / S and q[:, 0] += 2: the running row max rises with every chunk (at d = 128 by about
              5.7 nats over the sequence), so every chunk merge rescales.  The key offset (up to 32 in one dimension)
              also multiplies the rounding error of dQ = sigma sum_j dS_ij k_j (a sum that cancels): any attention that
              forms O from bf16 P in the forward has an intrinsic dQ error of 0.5-1.5e-2 here (R28, pinned
              on the CPU by tests/test_conditioning.py), so dQ is held to 3e-2 for this distribution and every other
              tensor to the 1e-2 bar;
  * extreme — q x 30: logits of +-100s of nats.  The running max jumps by tens of nats between chunks (past the
              kernels' lazy-rescale threshold of 8 in log2 units, R23), and most keys of a row sit more
              than 126 log2 units below its max, where exp2 underflows (both the MUFU path and the FMA-pipe
              polynomial, which clamps its argument at -126 so that it cannot wrap to NaN).

Each is checked against the fp64 oracle (normwise max relative error <= 1e-2 bf16, <= 1e-4 fp32) at d = 64 / 80 /
128, at world sizes 2 and 4 through the in-process group, under scheduler stress, and at the full configs[1] size on
sampled rows plus the dK / dV identities."""
import ctypes

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu

DISTS = ("drift32", "extreme")
DQ_TOL_DRIFT32 = 3e-2  # DESIGN.md R28


def _check(res, ref, tol, dist=None):
    errs = {n: rel_err(res[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(np.isfinite(res[n]).all() for n in errs), "non-finite output"
    bar = {n: (DQ_TOL_DRIFT32 if (n == "dq" and dist == "drift32" and tol > 1e-3) else tol) for n in errs}
    assert all(errs[n] <= bar[n] for n in errs), errs
    return errs


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("d", [64, 80, 128])
def test_bf16_extreme_logits(dist, d):
    x = inputs(dist, 61, 2048, 4, 2, d)            # u = 4 chunks of 512, GQA G = 2
    _check(run_cuda(x, 512, "bf16", 1), oracle_full(x), TOL["bf16"], dist)


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("d", [64, 80, 128])
def test_fp32_extreme_logits(dist, d):
    x = inputs(dist, 62, 1024, 2, 1, d)            # u = 4 chunks of 256
    _check(run_cuda(x, 256, "fp32", 1), oracle_full(x), TOL["fp32"])


@pytest.mark.parametrize("dist", DISTS)
def test_bf16_extreme_resident(dist):
    """offload = 0: one launch per query chunk over the whole resident key range (no chunk merge)."""
    x = inputs(dist, 63, 2048, 2, 2, 80)
    _check(run_cuda(x, 512, "bf16", 0), oracle_full(x), TOL["bf16"], dist)


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("p", [2, 4])
def test_multirank_extreme_logits(dist, p):
    from test_gpu_multirank import run_group
    S, Hq, Hkv, d, C = 2048, 8, 4, 80, 512
    x = gen.make_inputs(dist, 64, S, Hq, Hkv, d)
    got = run_group(x, p, C, "bf16", 1)
    _check(got, oracle_full(x), TOL["bf16"], dist)
    ref1 = run_group(x, 1, C, "bf16", 1)
    for n in ("o", "lse", "dk", "dv"):   # world-size invariance: bitwise
        assert np.array_equal(got[n], ref1[n]), n


@pytest.mark.parametrize("dist", DISTS)
def test_stress_extreme_logits(dist):
    from test_gpu_stress import _ctx, stressed
    S, Hq, Hkv, d, C = 2048, 8, 2, 80, 256
    x = inputs(dist, 65, S, Hq, Hkv, d)
    ctx = _ctx()
    base = run_cuda(x, C, "bf16", 1, ctx=ctx)
    ctx.close()
    with stressed(seed=5):
        ctx = _ctx()
        got = run_cuda(x, C, "bf16", 1, ctx=ctx)
        ctx.close()
    ref = oracle_full(x)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(got[n], base[n]), n
    assert rel_err(got["dq"], base["dq"]) < 2.0 ** -8
    _check(got, ref, TOL["bf16"], dist)


# ---------------------------------------------------------------------------------- configs[1] at full size
S_FULL, H_FULL, D_FULL, C_FULL = 524288, 32, 80, 65536


@pytest.fixture(scope="module", params=DISTS)
def full_run(request):
    from paper_2408_16978_b200 import _lib, fpdt
    dist = request.param
    torch.cuda.set_device(0)
    genlib = _lib.load_generator()
    S, H, D, C = S_FULL, H_FULL, D_FULL, C_FULL

    def gen_tensor(name):
        t = torch.empty(S, H, D, dtype=torch.bfloat16, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name], gen.DIST_IDS[dist],
                                  7, S, H, D, S, 0, 1, C, ctypes.c_void_p(0))
        assert rc == 0
        return t

    q, k, v, do = (gen_tensor(n) for n in ("q", "k", "v", "do"))
    o = torch.empty_like(q)
    lse = torch.empty(S, H, dtype=torch.float32, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ctx = fpdt.FPDTContext()
    fpdt.fpdt_attn_fwd(ctx, q, k, v, o, lse, S, H, H, D, 1, C, 1, fpdt.FPDT_BF16, 1)
    fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, H, H, D, 1, C, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    ctx.close()
    rng = np.random.default_rng(1)
    rows = sorted(set([0, S - 1] + [m * C for m in range(S // C)] + [m * C + C - 1 for m in range(S // C)]
                      + rng.integers(0, S, 8).tolist()))
    ridx = torch.tensor(rows, device="cuda")
    out = {
        "dist": dist, "rows": np.array(rows),
        "o": o.index_select(0, ridx).float().cpu().numpy(),
        "lse": lse.index_select(0, ridx).cpu().numpy(),
        "dq": dq.index_select(0, ridx).float().cpu().numpy(),
        "finite": bool(torch.isfinite(o).all() and torch.isfinite(dq).all() and torch.isfinite(dk).all()
                       and torch.isfinite(dv).all() and torch.isfinite(lse).all()),
        "dk_sum": dk.float().sum(0).cpu().numpy(), "dk_abs": dk.float().abs().sum(0).cpu().numpy(),
        "dv_sum": dv.float().sum(0).cpu().numpy(), "dv_abs": dv.float().abs().sum(0).cpu().numpy(),
        "do_sum": do.float().sum(0).cpu().numpy(),
    }
    del q, k, v, do, o, dq, dk, dv
    torch.cuda.empty_cache()
    return out


def test_fullsize_extreme_sampled_rows(full_run):
    from oracle import sampled
    S, H, D = S_FULL, H_FULL, D_FULL
    dist, rows = full_run["dist"], full_run["rows"]
    assert full_run["finite"]
    h = 9
    toks = np.arange(S)
    kg = gen.generate("k", dist, 7, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    vg = gen.generate("v", dist, 7, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    qr = gen.generate("q", dist, 7, rows, H, D, S, heads=[h])[:, 0]
    dor = gen.generate("do", dist, 7, rows, H, D, S, heads=[h])[:, 0]
    dq, o, lse = sampled.rows_dq(qr, dor, rows, kg, vg, sampled.default_scale(D))
    errs = {"o": rel_err(full_run["o"][:, h], o), "lse": rel_err(full_run["lse"][:, h], lse),
            "dq": rel_err(full_run["dq"][:, h], dq)}
    bar = {"o": TOL["bf16"], "lse": TOL["bf16"], "dq": DQ_TOL_DRIFT32 if dist == "drift32" else TOL["bf16"]}
    assert all(errs[n] <= bar[n] for n in errs), errs


def test_fullsize_extreme_identities(full_run):
    assert np.max(np.abs(full_run["dk_sum"]) / np.maximum(full_run["dk_abs"], 1e-30)) <= TOL["bf16"]
    assert np.max(np.abs(full_run["dv_sum"] - full_run["do_sum"]) / full_run["dv_abs"]) <= TOL["bf16"]
