#!/usr/bin/env python
"""Compute/exchange overlap of the p > 1 schedule on ONE GPU (SURVEY §8(a) stream/event skeleton).

p ranks of an in-process group (fpdt_group_create, one host thread and one stream per rank) run fpdt_attn_fwd +
fpdt_attn_bwd on the rank-ordinal shards of one global sequence.  Per rank, with the library's CUDA-event timing:
  step_ms      fwd + bwd on the rank's stream
  pair_ms      summed pair-kernel time
  gap_ms       time the compute stream spent between consecutive pair kernels of one call (waiting for an exchange,
               a host fetch or a support kernel; fpdt_kernel_gaps)
  a2a          the exchanges on the comm stream: count, total, first (pipeline fill) and last (drain), bytes
The claim under test: the exchanges overlap the pair kernels, so gap_ms stays near the unhidden fill/drain exchanges
(first + last) instead of growing with the number of chunks.  The local group's exchange is a copy-engine copy with
NCCL's layout (the ranks share one GPU, so kernels of different ranks also share the SMs).

    python tools/overlap_probe.py [--seq 131072] [--heads 32] [--dim 80] [--chunk 16384] [--p 2 4 8]
"""
import argparse
import ctypes
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fpdt_inputs as gen  # noqa: E402
from paper_2408_16978_b200 import _lib, fpdt  # noqa: E402


def run(p, S, H, d, C, offload, steps):
    s_local = S // p
    genlib = _lib.load_generator()
    group = fpdt.LocalGroup(p)
    out = [None] * p
    errors = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                def g(name):
                    t = torch.empty(s_local, H, d, dtype=torch.bfloat16, device="cuda")
                    assert genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name],
                                                gen.DIST_IDS["normal"], 0, s_local, H, d, S, r, p, C,
                                                ctypes.c_void_p(stream.cuda_stream)) == 0
                    return t
                q, k, v, do = g("q"), g("k"), g("v"), g("do")
                o, dq, dk, dv = (torch.empty_like(t) for t in (q, q, k, v))
            stream.synchronize()
            ctx = fpdt.FPDTContext(p, r, group=group)

            def step():
                fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, s_local, H, H, d, 1, C, p, fpdt.FPDT_BF16, offload, 0.0,
                                   stream)
                fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, s_local, H, H, d, 1, C, p, fpdt.FPDT_BF16, offload, 0.0,
                                   stream)
            step()
            stream.synchronize()
            ctx.set_kernel_timing(True)
            ctx.kernel_time(reset=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step()
            e1.record(stream)
            stream.synchronize()
            gap, ngap = ctx.kernel_gaps()
            x = ctx.exchange_time()
            f, nf, b, nb = ctx.kernel_time(reset=True)
            out[r] = {"rank": r, "step_ms": e0.elapsed_time(e1) / steps, "pair_ms": (f + b) / steps,
                      "gap_ms": gap / steps, "gaps": ngap // steps, "a2a_n": x["n"] // steps,
                      "a2a_total_ms": x["total_ms"] / steps, "a2a_first_ms": x["first_ms"], "a2a_last_ms": x["last_ms"],
                      "a2a_bytes": x["bytes"] // steps}
            ctx.close()
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(p)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    group.close()
    if errors:
        raise RuntimeError(errors)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--dim", type=int, default=80)
    ap.add_argument("--chunk", type=int, default=16384)
    ap.add_argument("--offload", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--p", type=int, nargs="+", default=[2, 4, 8])
    a = ap.parse_args()
    for p in a.p:
        ranks = run(p, a.seq, a.heads, a.dim, a.chunk, a.offload, a.steps)
        worst = max(ranks, key=lambda r: r["gap_ms"])
        rec = {"tool": "overlap_probe", "p": p, "S": a.seq, "heads": a.heads, "head_dim": a.dim, "chunk": a.chunk,
               "chunks": a.seq // a.chunk, "offload": a.offload, "ranks": ranks,
               "max_gap_ms": worst["gap_ms"], "fill_plus_drain_ms": worst["a2a_first_ms"] + worst["a2a_last_ms"],
               "a2a_total_ms": worst["a2a_total_ms"], "step_ms": max(r["step_ms"] for r in ranks)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
