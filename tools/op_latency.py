#!/usr/bin/env python
"""B200 op-latency study (fig:avg_time): per chunk length s, the time of
  - attention forward / backward on a [s, h/p, d] chunk (the library's tcgen05 pair kernels via fpdt_debug_pair):
    the causal diagonal block (the paper's "attention on [b, s, h/p, d]") and a full (unmasked) chunk pair, which is
    what FPDT's pipeline overlaps with each fetch;
  - host-to-device fetching of [3, s, h/p, d] bf16 (q, k, v: the paper's fetch unit) from pinned memory, and of the
    units the library actually moves: the forward's key/value chunk [2, s, hkv, d] and the backward's query-side set
    (q, dO bf16 + fp32 dq partial);
on ONE B200 (the all-to-all and the one-GPU-fetches-and-scatters strategy need several GPUs: not measured here).
The crossover the paper reports at 32K-64K on A100 is where attention overtakes the fetch.

    python tools/op_latency.py [--heads 4] [--d 80] [--lens 4096 ... 262144]
Prints one JSON line per chunk length.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_16978_b200 import _lib  # noqa: E402


def ev_time(fn, reps, stream=None):
    stream = stream or torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=4, help="q heads per rank (h/p); 32 heads at p = 8 -> 4")
    ap.add_argument("--kv-heads", type=int, default=0, help="kv heads per rank (0 = --heads)")
    ap.add_argument("--d", type=int, default=80)
    ap.add_argument("--lens", type=int, nargs="+",
                    default=[4096, 8192, 16384, 32768, 65536, 131072, 262144])
    args = ap.parse_args()
    H, d = args.heads, args.d
    Hkv = args.kv_heads or H
    lib = _lib.load_diag()
    P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    bf = torch.bfloat16
    torch.manual_seed(0)
    for s in args.lens:
        q, do = (torch.randn(s, H, d, device="cuda").to(bf) for _ in range(2))
        k, v = (torch.randn(s, Hkv, d, device="cuda").to(bf) for _ in range(2))
        o = torch.empty_like(q)
        lse2 = torch.empty(H, s, device="cuda")
        Dst = torch.zeros(H, s, device="cuda")
        dq = torch.zeros(H, s, d, device="cuda")
        dk, dv = torch.empty_like(k), torch.empty_like(v)
        res = {"s": s, "heads_q": H, "heads_kv": Hkv, "head_dim": d}
        for causal in (1, 0):
            def fwd():
                rc = lib.fpdt_debug_pair(0, d, causal, P(q), P(k), P(v), None, None, None, P(o), P(lse2), None, s, H,
                                         Hkv, None, 0, None)
                assert rc == 0, rc

            def bwd():
                rc = lib.fpdt_debug_pair(1, d, causal, P(q), P(k), P(v), P(do), P(lse2), P(Dst), P(dq), P(dk), P(dv),
                                         s, H, Hkv, None, 0, None)
                assert rc == 0, rc

            reps = max(2, min(50, int(2 ** 34 / (s * s))))
            fwd()  # lse2 of this block for the backward
            tf, tb = ev_time(fwd, reps), ev_time(bwd, reps)
            pairs = s * (s + 1) / 2 if causal else s * s
            tag = "diag" if causal else "full"
            res[f"attn_fwd_{tag}_ms"] = tf
            res[f"attn_bwd_{tag}_ms"] = tb
            res[f"attn_fwd_{tag}_tflops"] = 4 * d * H * pairs / tf / 1e9
            res[f"attn_bwd_{tag}_tflops"] = 10 * d * H * pairs / tb / 1e9
        # host-to-device fetches from pinned memory on a copy stream (CUDA events on that stream)
        cp = torch.cuda.Stream()
        units = {"qkv": 3 * s * H * d * 2, "kv_fwd": 2 * s * Hkv * d * 2, "q_side_bwd": s * H * d * (2 + 2 + 4)}
        for name, nbytes in units.items():
            h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            with torch.cuda.stream(cp):
                t = ev_time(lambda: dev.copy_(h, non_blocking=True), 5, cp)
            res[f"h2d_{name}_ms"] = t
            res[f"h2d_{name}_GBps"] = nbytes / t / 1e6
            del h, dev
        res["attn_fwd_diag_over_h2d_qkv"] = res["attn_fwd_diag_ms"] / res["h2d_qkv_ms"]
        res["pair_fwd_over_kv_fetch"] = res["attn_fwd_full_ms"] / res["h2d_kv_fwd_ms"]
        res["pair_bwd_over_q_side_fetch"] = res["attn_bwd_full_ms"] / res["h2d_q_side_bwd_ms"]
        print(json.dumps(res), flush=True)
        del q, k, v, do, o, lse2, Dst, dq, dk, dv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
