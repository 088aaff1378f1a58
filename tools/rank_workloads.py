#!/usr/bin/env python
"""Per-rank attention workloads of BASELINE.json configs[2..4] on ONE B200.

After the sequence-to-head all-to-all, rank r of a p-GPU Ulysses run computes chunked causal attention over the
WHOLE sequence S for its Hq/p query heads and Hkv/p kv heads.  That per-rank
work — every chunk pair, offload and prefetch included — is exactly a p = 1 call with Hq/p and Hkv/p heads, which
is what this tool runs.  Only the all-to-alls are missing (one B200 on this pool), so the numbers are the
per-GPU compute + host-offload part of the multi-GPU configs, not a multi-GPU measurement.

    python tools/rank_workloads.py [--only c2p1 c2p8 c3 c4 c5] [--steps 1]

Prints one JSON line per (config, chunk): step seconds (CUDA events), pair-kernel seconds, TFLOPS/GPU,
host bytes and host-link GB/s, device and pinned-host footprint.
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

K = 1024
M = 1024 * 1024
# (name, BASELINE.json config text, S, Hq, Hkv, d, p, chunks)
WORKLOADS = [
    # configs[1] (GPT-2.7B, 32 heads x 80, S = 512K, C = 64K) per rank at p = 1, 2, 4, 8: the compute side of its
    # strong scaling (the all-to-alls excluded)
    ("c2p1", "GPT-2.7B layer (32 heads, d=80), S=512K, one GPU", 512 * K, 32, 32, 80, 1, [64 * K]),
    ("c2p2", "GPT-2.7B layer (32 heads, d=80), S=512K across 2 GPUs", 512 * K, 32, 32, 80, 2, [64 * K]),
    ("c2p4", "GPT-2.7B layer (32 heads, d=80), S=512K across 4 GPUs", 512 * K, 32, 32, 80, 4, [64 * K]),
    ("c2p8", "GPT-2.7B layer (32 heads, d=80), S=512K across 8 GPUs", 512 * K, 32, 32, 80, 8, [64 * K]),
    ("c3", "Llama-3 8B layer (32 q / 8 kv heads, d=128), S=2M across 4 GPUs, host-offloaded KV", 2 * M, 32, 8, 128,
     4, [64 * K]),
    ("c4", "13B layer (40 heads, d=128), S=4M across 8 GPUs, chunk-size sweep 32K-256K", 4 * M, 40, 40, 128, 8,
     [32 * K, 64 * K, 128 * K, 256 * K]),
    ("c5", "70B layer (64 q / 8 kv heads, d=128), S=1M across 8 GPUs, offload + prefetch", 1 * M, 64, 8, 128, 8,
     [64 * K]),
]


def run_one(name, text, S, Hq, Hkv, d, p, C, steps, genlib, bwd_order=0):
    hq, hkv = Hq // p, Hkv // p
    rec = {"config": name, "text": text, "S": S, "world_size_emulated": p, "heads_q_per_rank": hq,
           "heads_kv_per_rank": hkv, "head_dim": d, "chunk": C, "chunks": S // C, "offload": 1}

    def gen_tensor(tname, h):
        t = torch.empty(S, h, d, dtype=torch.bfloat16, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[tname], gen.DIST_IDS["normal"],
                                  0, S, h, d, S, 0, 1, C, ctypes.c_void_p(0))
        assert rc == 0
        return t

    q, k, v, do = gen_tensor("q", hq), gen_tensor("k", hkv), gen_tensor("v", hkv), gen_tensor("do", hq)
    o = torch.empty_like(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ctx = fpdt.FPDTContext()
    ctx.set_kernel_timing(True)
    ctx.set_bwd_order(bwd_order)
    stream = torch.cuda.current_stream()
    times = []
    for s in range(steps):
        ctx.kernel_time(reset=True)
        st0 = ctx.stats()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(stream)
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S, hq, hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1, 0.0, stream)
        fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, hq, hkv, d, 1, C, 1, fpdt.FPDT_BF16, 1, 0.0, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        st1 = ctx.stats()
        fwd_ms, n_fwd, bwd_ms, n_bwd = ctx.kernel_time(reset=True)
        times.append((e0.elapsed_time(e1) / 1e3, wall, fwd_ms / 1e3, bwd_ms / 1e3, n_fwd, n_bwd,
                      st1["bytes_h2d"] - st0["bytes_h2d"], st1["bytes_d2h"] - st0["bytes_d2h"]))
    dt, wall, fwd_s, bwd_s, n_fwd, n_bwd, h2d, d2h = times[-1]
    flops = 14 * d * hq * S * (S + 1) / 2
    st = ctx.stats()
    ok = bool(torch.isfinite(dq[-1].float()).all() and torch.isfinite(o[-1].float()).all()
              and torch.isfinite(dk[0].float()).all())
    rec.update(ok=ok, steps=steps, timed_step="last", step_s=dt, wall_s=wall, fwd_kernel_s=fwd_s, bwd_kernel_s=bwd_s,
               fwd_launches=n_fwd, bwd_launches=n_bwd,
               tflops_per_gpu=flops / dt / 1e12, fwd_kernel_tflops=4 * d * hq * S * (S + 1) / 2 / fwd_s / 1e12,
               bwd_kernel_tflops=10 * d * hq * S * (S + 1) / 2 / bwd_s / 1e12,
               tokens_per_s_p_gpus=S / dt, h2d_bytes=h2d, d2h_bytes=d2h, h2d_GBps=h2d / dt / 1e9,
               d2h_GBps=d2h / dt / 1e9, device_bytes_caller=sum(t.numel() * 2 for t in (q, k, v, do, o, dq, dk, dv)),
               device_bytes_library=st["device_bytes"], host_pinned_bytes=st["host_arena_bytes"],
               first_step_s=times[0][0],
               # Q-outer runs two pair kernels at a time on two streams: the summed per-launch times then overlap
               # and the *_kernel_tflops fields undercount; step_s is the measure
               concurrent_pairs=st["bwd_order"] == 1 and os.environ.get("FPDT_BWD_QO_STREAMS", "2") != "1", bwd_order=["kv_outer", "q_outer"][st["bwd_order"]],
               host_dkv_pinned_bytes=st["host_dkv_bytes"])
    ctx.close()
    del q, k, v, do, o, dq, dk, dv
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="+", default=None)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--chunks", type=int, nargs="+", default=None, help="restrict the chunk sizes (in K tokens)")
    ap.add_argument("--bwd-order", default="kv", choices=["kv", "q", "auto"],
                    help="backward loop order (fpdt_set_bwd_order)")
    args = ap.parse_args()
    order = {"kv": fpdt.FPDT_BWD_KV_OUTER, "q": fpdt.FPDT_BWD_Q_OUTER, "auto": fpdt.FPDT_BWD_AUTO}[args.bwd_order]
    torch.cuda.set_device(0)
    genlib = _lib.load_generator()
    for name, text, S, Hq, Hkv, d, p, chunks in WORKLOADS:
        if args.only and name not in args.only:
            continue
        for C in chunks:
            if args.chunks and C // K not in args.chunks:
                continue
            try:
                rec = run_one(name, text, S, Hq, Hkv, d, p, C, args.steps, genlib, order)
            except Exception as e:  # report and continue with the next workload
                rec = {"config": name, "chunk": C, "ok": False, "error": f"{type(e).__name__}: {str(e)[:200]}"}
                torch.cuda.empty_cache()
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
