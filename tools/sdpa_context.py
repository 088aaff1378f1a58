#!/usr/bin/env python
"""Context comparison (optional): the box's PyTorch SDPA backends on one causal chunk pair of the bench
shape (one 65,536-token chunk, 32 heads, d = 80, bf16), fwd + bwd, against this library's pair kernels on the same
shape (fpdt_debug_pair, the diagonal pair).  Same FLOP convention (causal pairs x (4d fwd + 10d bwd) per head).
Library kernels, not the bar: the reference has no Blackwell kernel.

    python tools/sdpa_context.py [--seq 65536] [--heads 32] [--dim 80]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=65536)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=80)
    a = ap.parse_args()
    S, H, d = a.seq, a.heads, a.dim
    pairs = S * (S + 1) / 2
    f_fwd, f_bwd = 4 * d * H * pairs, 10 * d * H * pairs
    torch.manual_seed(0)
    q, k, v, do = (torch.randn(1, H, S, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    out = []
    for name, be in (("flash", SDPBackend.FLASH_ATTENTION), ("cudnn", SDPBackend.CUDNN_ATTENTION),
                     ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
        try:
            qq, kk, vv = (t.detach().clone().requires_grad_(True) for t in (q, k, v))
            with sdpa_kernel(be):
                fwd_ms = timed(lambda: F.scaled_dot_product_attention(qq, kk, vv, is_causal=True))
                o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)

                def fb():
                    y = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                    y.backward(do)
                fb_ms = timed(fb)
            del o
            out.append({"impl": f"torch sdpa {name}", "fwd_ms": fwd_ms, "bwd_ms": fb_ms - fwd_ms,
                        "fwd_tflops": f_fwd / fwd_ms / 1e9, "bwd_tflops": f_bwd / (fb_ms - fwd_ms) / 1e9})
        except Exception as e:  # noqa: BLE001
            out.append({"impl": f"torch sdpa {name}", "error": str(e)[:160]})
    # this library's pair kernels on the same data (layout [S][H][d])
    from paper_2408_16978_b200 import fpdt
    lib = fpdt.diag()
    qs, ks, vs, dos = (t[0].transpose(0, 1).contiguous() for t in (q, k, v, do))
    o = torch.empty_like(qs)
    lse2 = torch.empty(H, S, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    fwd_ms = timed(lambda: lib.fpdt_debug_pair(0, d, 1, P(qs), P(ks), P(vs), None, None, None, P(o), P(lse2), None, S,
                                               H, H, None, 0, None))
    Dst = torch.zeros(H, S, device="cuda")
    dq = torch.zeros(H, S, d, device="cuda")
    dk, dv = torch.empty_like(ks), torch.empty_like(vs)
    bwd_ms = timed(lambda: lib.fpdt_debug_pair(1, d, 1, P(qs), P(ks), P(vs), P(dos), P(lse2), P(Dst), P(dq), P(dk),
                                               P(dv), S, H, H, None, 0, None))
    out.append({"impl": "fpdt (this library) pair kernels", "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                "fwd_tflops": f_fwd / fwd_ms / 1e9, "bwd_tflops": f_bwd / bwd_ms / 1e9})
    for r in out:
        r.update({"tool": "sdpa_context", "S": S, "heads": H, "head_dim": d, "causal": True})
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
