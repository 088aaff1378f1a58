#!/usr/bin/env python
"""Attention block with the fused QKV projection (fpdt_block_fwd/bwd) against the attention-only
calls at the GPT-2.7B shape of BASELINE.json configs[1] on one B200: hidden 2560 = 32 heads x 80, S = 512K,
C = 64K, offload on.  Same random bf16 data for both (torch.randn, seed 0; a timing tool, parity is in
tests/test_gpu_block.py).  CUDA-event timing on the caller's stream, W warm-up steps, K timed steps.

    python tools/block_bench.py [--seq 524288] [--steps 2] [--warmup 1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_16978_b200 import fpdt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    S, C, H, d = args.seq, args.chunk, 32, 80
    hidden, N = H * d, 3 * H * d
    torch.manual_seed(0)
    bf = torch.bfloat16
    x = torch.randn(S, hidden, dtype=bf, device="cuda")
    w = (torch.randn(hidden, N, dtype=bf, device="cuda") * (hidden ** -0.5)).to(bf)
    do = torch.randn(S, H, d, dtype=bf, device="cuda")
    with torch.no_grad():
        qkv = (x @ w).view(S, 3, H, d)
        q, k, v = (qkv[:, i].contiguous() for i in range(3))
        del qkv
    o = torch.empty(S, H, d, dtype=bf, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dx = torch.empty_like(x)
    dw = torch.empty(hidden, N, dtype=torch.float32, device="cuda")
    wo = (torch.randn(H * d, hidden, dtype=bf, device="cuda") * ((H * d) ** -0.5)).to(bf)
    y = torch.empty(S, hidden, dtype=bf, device="cuda")
    dy = torch.randn(S, hidden, dtype=bf, device="cuda")
    dwo = torch.empty(H * d, hidden, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    B = fpdt.FPDT_BF16
    ctx = fpdt.FPDTContext()

    def attn_step():
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, H, d, 1, C, 1, B, 1, 0.0, stream)
        fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, H, H, d, 1, C, 1, B, 1, 0.0, stream)

    def block_step():
        fpdt.fpdt_block_fwd(ctx, x, w, o, None, S, hidden, H, H, d, 1, C, 1, B, 1, 0.0, stream)
        fpdt.fpdt_block_bwd(ctx, x, w, o, do, dx, dw, S, hidden, H, H, d, 1, C, 1, B, 1, 0.0, stream)

    def block_o_step():
        fpdt.fpdt_block_fwd(ctx, x, w, o, None, S, hidden, H, H, d, 1, C, 1, B, 1, 0.0, stream, w_o=wo, y=y)
        fpdt.fpdt_block_bwd(ctx, x, w, o, dy, dx, dw, S, hidden, H, H, d, 1, C, 1, B, 1, 0.0, stream, w_o=wo,
                            dw_o=dwo)

    def timed(step):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st0 = ctx.stats()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        st1 = ctx.stats()
        return e0.elapsed_time(e1) / args.steps / 1e3, (st1["kernel_launches"] - st0["kernel_launches"]) // args.steps

    t_attn, l_attn = timed(attn_step)
    t_block, l_block = timed(block_step)
    t_block_o, l_block_o = timed(block_o_step)
    f_attn = 14 * d * H * S * (S + 1) / 2
    f_proj = 6 * S * hidden * N  # fwd x W, bwd dx = dqkv W^T and dW = x^T dqkv
    rec = {"tool": "block_bench", "S": S, "chunk": C, "heads": H, "head_dim": d, "hidden": hidden, "offload": 1,
           "steps": args.steps, "attn_step_s": t_attn, "block_step_s": t_block,
           "projection_overhead_s": t_block - t_attn, "projection_flops": f_proj,
           "attn_tflops": f_attn / t_attn / 1e12, "block_tflops": (f_attn + f_proj) / t_block / 1e12,
           "block_tokens_per_s": S / t_block, "attn_tokens_per_s": S / t_attn,
           "launches_attn": l_attn, "launches_block": l_block,
           "block_with_out_proj_step_s": t_block_o, "out_proj_flops": 6 * S * hidden * H * d,
           "block_with_out_proj_tflops": (f_attn + f_proj + 6 * S * hidden * H * d) / t_block_o / 1e12,
           "launches_block_with_out_proj": l_block_o, "dwo_finite": bool(torch.isfinite(dwo).all()),
           "dx_finite": bool(torch.isfinite(dx).all()), "dw_finite": bool(torch.isfinite(dw).all())}
    print(json.dumps(rec), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
