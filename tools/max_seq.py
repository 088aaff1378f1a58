#!/usr/bin/env python
"""Maximum sequence length sustained on ONE B200 (BASELINE.json north_star: "the maximum sequence length sustained
per GPU"): one full fwd+bwd step through the C-ABI with host-offloaded KV chunks, at growing S, until the device or
the pinned host store runs out (or --max-s is reached).

    python tools/max_seq.py [--heads 32 --kv-heads 32 --d 80 --chunk 65536] [--s 1048576 2097152 3145728]

Prints one JSON line per S: step seconds, TFLOPS, device bytes (caller tensors + library working set), pinned host
bytes, or the error that stopped the sweep.
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fpdt_inputs as gen  # noqa: E402
from paper_2408_16978_b200 import _lib, fpdt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--d", type=int, default=80)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--s", type=int, nargs="+", default=[1 << 20, 2 << 20, 3 << 20])
    ap.add_argument("--steps", type=int, default=1, help="steps per length (the first includes pinned allocation)")
    ap.add_argument("--bwd-order", default="kv", choices=["kv", "q", "auto"])
    args = ap.parse_args()
    torch.cuda.set_device(0)
    genlib = _lib.load_generator()
    H, Hkv, d, C = args.heads, args.kv_heads, args.d, args.chunk
    for S in args.s:
        rec = {"S": S, "heads_q": H, "heads_kv": Hkv, "head_dim": d, "chunk": C, "offload": 1}
        try:
            def gen_tensor(name, h):
                t = torch.empty(S, h, d, dtype=torch.bfloat16, device="cuda")
                rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name],
                                          gen.DIST_IDS["normal"], 0, S, h, d, S, 0, 1, C, ctypes.c_void_p(0))
                assert rc == 0
                return t
            q, k, v, do = gen_tensor("q", H), gen_tensor("k", Hkv), gen_tensor("v", Hkv), gen_tensor("do", H)
            o = torch.empty_like(q)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            ctx = fpdt.FPDTContext()
            ctx.set_bwd_order({"kv": 0, "q": 1, "auto": 2}[args.bwd_order])
            steps = []
            for _ in range(args.steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, H, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
                fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, H, Hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1)
                torch.cuda.synchronize()
                steps.append(time.perf_counter() - t0)
            dt = steps[-1]
            st = ctx.stats()
            flops = 14 * d * H * S * (S + 1) / 2
            ok = bool(torch.isfinite(dq[-1].float()).all() and torch.isfinite(o[-1].float()).all())
            rec.update(ok=ok, steps_s=steps, bwd_order=["kv_outer", "q_outer"][st["bwd_order"]],
                       host_dkv_pinned_bytes=st["host_dkv_bytes"], step_s=dt, tflops=flops / dt / 1e12, tokens_per_s=S / dt,
                       device_bytes_caller=sum(t.numel() * 2 for t in (q, k, v, do, o, dq, dk, dv)),
                       device_bytes_library=st["device_bytes"], host_pinned_bytes=st["host_arena_bytes"])
            ctx.close()
            del q, k, v, do, o, dq, dk, dv
            torch.cuda.empty_cache()
        except Exception as e:  # OOM (device or pinned host) ends the sweep
            rec.update(ok=False, error=f"{type(e).__name__}: {str(e)[:200]}")
            print(json.dumps(rec), flush=True)
            break
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
