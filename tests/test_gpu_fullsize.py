"""Parity at BASELINE.json's full size, in the launch configuration bench.py times.

configs[1] (the bench workload): GPT-2.7B-shaped layer, S = 524,288, 32 heads, head_dim 80, chunk 65,536
(u = 8), bf16, causal, offload ON, world size 1 — the same seeded inputs (device generator, distribution
"normal", seed 0) and the same C-ABI calls as bench.py.  The oracle cannot run the whole sequence, so
(SURVEY §8(c) c.5):
  * sampled rows: O, lse and dQ of rows at every chunk boundary (first/last row of each chunk), the first and
    last row of the sequence and seeded random rows, for two heads, against oracle/sampled.rows_dq (fp64,
    the plain definition restricted to one row);
  * tail columns: dK, dV of the last 128 key positions of one head against oracle/sampled.tail_dkdv;
  * identities on the FULL dK / dV of every head: sum_j dK_j = 0 and sum_j dV_j = sum_i dO_i (rows of P sum
    to 1, and sum_j dS_ij = 0), which hold for the exact gradient at any size.
Bar: normwise max relative error <= 1e-2 (north_star, bf16 I/O with fp32 accumulation)."""
import ctypes

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, rel_err
from oracle import sampled

pytestmark = pytest.mark.gpu

S, H, D, C = 524288, 32, 80, 65536
HEADS = (0, 17)


@pytest.fixture(scope="module")
def run():
    from paper_2408_16978_b200 import _lib, fpdt
    torch.cuda.set_device(0)
    genlib = _lib.load_generator()

    def gen_tensor(name):
        t = torch.empty(S, H, D, dtype=torch.bfloat16, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name], gen.DIST_IDS["normal"],
                                  0, S, H, D, S, 0, 1, C, ctypes.c_void_p(0))
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
    st = ctx.stats()
    ctx.close()
    rng = np.random.default_rng(0)
    rows = sorted(set([0, S - 1] + [m * C for m in range(S // C)] + [m * C + C - 1 for m in range(S // C)]
                      + rng.integers(0, S, 12).tolist()))
    ridx = torch.tensor(rows, device="cuda")
    out = {
        "rows": np.array(rows),
        "o": o.index_select(0, ridx).float().cpu().numpy(),
        "lse": lse.index_select(0, ridx).cpu().numpy(),
        "dq": dq.index_select(0, ridx).float().cpu().numpy(),
        "dk_tail": dk[S - 128:].float().cpu().numpy(),
        "dv_tail": dv[S - 128:].float().cpu().numpy(),
        # identities, reduced on the device over all S rows (fp32 sums of the bf16 outputs)
        "dk_sum": dk.float().sum(0).cpu().numpy(), "dk_abs": dk.float().abs().sum(0).cpu().numpy(),
        "dv_sum": dv.float().sum(0).cpu().numpy(), "dv_abs": dv.float().abs().sum(0).cpu().numpy(),
        "do_sum": do.float().sum(0).cpu().numpy(),
        "stats": st,
    }
    del q, k, v, do, o, dq, dk, dv
    torch.cuda.empty_cache()
    return out


def _head_inputs(h, rows):
    """Oracle-side regeneration (numpy twin) of what one head sees: all keys/values, the sampled q/dO rows."""
    toks = np.arange(S)
    kg = gen.generate("k", "normal", 0, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    vg = gen.generate("v", "normal", 0, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    qr = gen.generate("q", "normal", 0, rows, H, D, S, heads=[h])[:, 0]
    dor = gen.generate("do", "normal", 0, rows, H, D, S, heads=[h])[:, 0]
    return kg, vg, qr, dor


@pytest.mark.parametrize("h", HEADS)
def test_fullsize_sampled_rows(run, h):
    rows = run["rows"]
    kg, vg, qr, dor = _head_inputs(h, rows)
    dq, o, lse = sampled.rows_dq(qr, dor, rows, kg, vg, sampled.default_scale(D))
    errs = {"o": rel_err(run["o"][:, h], o), "lse": rel_err(run["lse"][:, h], lse),
            "dq": rel_err(run["dq"][:, h], dq)}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_fullsize_tail_columns(run):
    h = 5
    T = 128
    toks = np.arange(S)
    kg = gen.generate("k", "normal", 0, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    vg = gen.generate("v", "normal", 0, toks, H, D, S, heads=[h])[:, 0].astype(np.float64)
    tail = np.arange(S - T, S)
    qt = gen.generate("q", "normal", 0, tail, H, D, S, heads=[h])[:, 0][None]
    dot = gen.generate("do", "normal", 0, tail, H, D, S, heads=[h])[:, 0][None]
    dk, dv = sampled.tail_dkdv(qt, dot, S - T, kg, vg, sampled.default_scale(D))
    errs = {"dk": rel_err(run["dk_tail"][:, h], dk), "dv": rel_err(run["dv_tail"][:, h], dv)}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs


def test_fullsize_gradient_identities(run):
    # |sum_j dK_j| against sum_j |dK_j|, per head and dimension; sum_j dV_j = sum_i dO_i likewise
    assert np.max(np.abs(run["dk_sum"]) / run["dk_abs"]) <= TOL["bf16"]
    assert np.max(np.abs(run["dv_sum"] - run["do_sum"]) / run["dv_abs"]) <= TOL["bf16"]


def test_fullsize_offload_schedule(run):
    st = run["stats"]
    assert st["fetch_slots_highwater"] <= 2
    u = S // C
    kv_chunk = C * 2 * H * D * 2
    q_chunk = C * H * D * 2
    fwd_h2d = sum(range(u)) * kv_chunk
    bwd_h2d = u * kv_chunk + sum(u - j for j in range(u)) * 2 * q_chunk + sum(u - j for j in range(1, u)) * C * H * D * 4
    assert st["bytes_h2d"] == fwd_h2d + bwd_h2d
