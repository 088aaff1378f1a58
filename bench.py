#!/usr/bin/env python
"""FPDT chunked, sequence-parallel causal attention fwd+bwd on B200: the BASELINE.json headline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--offload 0|1]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...     (N > 1)

Workload (BASELINE.json configs[1]): GPT-2.7B-shaped attention layer, 32 heads, head_dim 80, global
sequence S = 524,288 tokens, chunk 65,536 (u = 8 / p chunks per rank), bf16, causal, one process per GPU,
Ulysses all-to-all per chunk for N > 1 (strong scaling: S fixed, s_local = S / N), KV chunks offloaded to
pinned host memory and prefetched back double-buffered (the paper's FPDT with offloading).
A step = fpdt_attn_fwd + fpdt_attn_bwd over the whole sequence.  Inputs are synthetic (the seeded
counter-based generator, distribution "normal"), resident in HBM; every input tensor is 2.7 GB (> 126 MB
L2), so no L2 flush is needed between steps.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunked attn fwd+bwd TFLOPS/GPU & tokens/s at 1/2/4/8 B200 vs bf16 peak"
WORKLOAD = dict(name="GPT-2.7B-shaped causal attention layer (BASELINE.json configs[1])", S=524288, Hq=32, Hkv=32,
                d=80, C=65536, dtype="bf16")


def flops_per_step(S, Hq, d, keep=None, C=None):
    pairs = S * (S + 1) / 2  # causal (query, key) pairs incl. the diagonal
    if keep is not None:  # block-sparse (§5.6): only the kept chunk blocks are computed
        u = keep.shape[0]
        pairs = u * C * (C + 1) / 2 + float(np.tril(keep, -1).sum()) * C * C
    return 4 * d * Hq * pairs, 10 * d * Hq * pairs  # fwd (QK^T, PV), bwd (recompute QK^T, dP, dV, dK, dQ)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p.get("bf16_tflops"), p.get("bf16_tflops_sustained"), p.get("hbm_gbs"), "measured (MEASURED_PEAKS.json)"
    return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def max_seq_record():
    """The longest sequence one B200 sustained through the C-ABI (fwd + bwd, offload on), from the committed
    tools/max_seq.py runs (a separate multi-minute job, not repeated inside this bench)."""
    best = None
    for name in ("r02_max_seq.jsonl", "r01_max_seq.jsonl", "r01_max_seq_8b_v2.jsonl"):
        path = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(path):
            continue
        with open(path) as f:
            for line in f:
                try:
                    r = json.loads(line)
                except ValueError:
                    continue
                S = r.get("S") or r.get("seq")
                if S and (best is None or S > best["tokens"]):
                    best = {"tokens": S, "shape": {k: r.get(k) for k in ("heads_q", "heads_kv", "head_dim", "chunk")
                                                   if k in r}, "step_s": r.get("step_s"), "source": f"profiles/{name}"}
    return best


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------------------ CPU oracle
def oracle_sample(S_sample=4096, heads=2, d=80, seed=0):
    """One bounded sample of the workload through the fp64 oracle (plain definition, fwd + bwd):
    the first S_sample tokens of `heads` heads.  Returns (seconds, algorithmic FLOPs of the sample)."""
    import fpdt_inputs as gen
    from oracle import attention
    x = gen.make_inputs("normal", seed, S_sample, heads, heads, d)
    t0 = time.perf_counter()
    o, lse = attention.attention_forward(x["q"], x["k"], x["v"])
    attention.attention_backward(x["q"], x["k"], x["v"], o, lse, x["do"])
    dt = time.perf_counter() - t0
    f, b = flops_per_step(S_sample, heads, d)
    return dt, f + b


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def projected_tokens_per_s(dt, sample_flops, S, Hq, d):
    f, b = flops_per_step(S, Hq, d)
    return S / (dt * (f + b) / sample_flops)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    W = WORKLOAD
    S, Hq, d = W["S"], W["Hq"], W["d"]
    sample = dict(S_sample=4096, heads=2, d=d)
    for _ in range(args.warmup):
        oracle_sample(**sample)
    times, fl = [], None
    for _ in range(args.steps):
        dt, fl = oracle_sample(**sample)
        times.append(dt)
    t = sum(times) / len(times)
    value = projected_tokens_per_s(t, fl, S, Hq, d)
    desc = (f"fp64 numpy oracle (oracle/attention.py), fwd+bwd of the first {sample['S_sample']} tokens x "
            f"{sample['heads']} heads (d={d}) per step; projected to the full workload by algorithmic FLOPs")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": W["name"], "S": S, "heads": Hq, "head_dim": d, "chunk": W["C"]},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------ ours
def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2408_16978_b200 import _lib, distributed, fpdt
    import fpdt_inputs as gen

    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    distributed.init_process_group(rank, world, "gloo")
    W = WORKLOAD
    S, Hq, Hkv, d, C = W["S"], W["Hq"], W["Hkv"], W["d"], W["C"]
    if args.seq:
        S = args.seq
    if args.chunk:
        C = args.chunk
    s_local = S // world
    offload = args.offload

    # NCCL id through torch.distributed (plumbing only)
    nid = distributed.broadcast_nccl_id(rank, world, fpdt.fpdt_get_unique_id)
    if world == 1 and args.exchange_path:
        nid = fpdt.fpdt_get_unique_id()  # one-rank communicator: the world-size > 1 schedule with NCCL self-exchanges
    ctx = fpdt.FPDTContext(world, rank, nid, local)
    if args.residency:
        ctx.set_residency(*args.residency)
    ctx.set_bwd_order({"kv": fpdt.FPDT_BWD_KV_OUTER, "q": fpdt.FPDT_BWD_Q_OUTER, "auto": fpdt.FPDT_BWD_AUTO}[args.bwd_order])
    keep = None
    if args.sparsity > 0:
        keep = gen.sparsity_plan(S // C, args.sparsity, seed=0)
        ctx.set_sparsity(keep)
    genlib = _lib.load_generator()
    bf = torch.bfloat16

    def gen_tensor(name, H):
        t = torch.empty(s_local, H, d, dtype=bf, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name], gen.DIST_IDS["normal"],
                                  0, s_local, H, d, S, rank, world, C, ctypes.c_void_p(0))
        assert rc == 0
        return t

    q, k, v, do = gen_tensor("q", Hq), gen_tensor("k", Hkv), gen_tensor("v", Hkv), gen_tensor("do", Hq)
    o = torch.empty_like(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    stream = torch.cuda.current_stream()

    def step():
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, s_local, Hq, Hkv, d, 1, C, world, fpdt.FPDT_BF16, offload,
                           0.0, stream)
        fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, s_local, Hq, Hkv, d, 1, C, world, fpdt.FPDT_BF16, offload,
                           0.0, stream)

    def barrier():
        distributed.barrier(world)

    def max_over_ranks(x):
        return distributed.max_over_ranks(x, world)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---------------------------------------------------------------- device-timed region
    ctx.set_kernel_timing(not args.no_kernel_timing)
    ctx.kernel_time(reset=True)
    st0 = ctx.stats()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.5)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    st1 = ctx.stats()
    gap_ms, n_gaps = ctx.kernel_gaps()
    xch = ctx.exchange_time()
    fwd_ms, n_fwd, bwd_ms, n_bwd = ctx.kernel_time(reset=True)
    ctx.set_kernel_timing(False)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = (st1["kernel_launches"] - st0["kernel_launches"]) // args.steps
    h2d_lib = (st1["bytes_h2d"] - st0["bytes_h2d"]) // args.steps
    d2h_lib = (st1["bytes_d2h"] - st0["bytes_d2h"]) // args.steps

    f_fwd, f_bwd = flops_per_step(S, Hq, d, keep, C)
    tokens_per_s = S / (ms / 1e3)
    tflops_gpu = (f_fwd + f_bwd) / (world * ms / 1e3) / 1e12
    burst, sustained, hbm, peak_src = load_peaks()

    # dominant kernel = the backward pair kernel (10d of the 14d FLOPs per pair); algorithmic FLOPs per launch
    # = (bwd FLOPs of a step / launches per step), timed by CUDA events on its launch stream inside the steps
    bwd_launch_ms = bwd_ms / max(n_bwd, 1)
    fwd_launch_ms = fwd_ms / max(n_fwd, 1)
    bwd_flops_launch = f_bwd / world / max(n_bwd // args.steps, 1)
    fwd_flops_launch = f_fwd / world / max(n_fwd // args.steps, 1)
    ach_bwd = bwd_flops_launch / (bwd_launch_ms / 1e3) / 1e12 if bwd_launch_ms > 0 else float("nan")
    ach_fwd = fwd_flops_launch / (fwd_launch_ms / 1e3) / 1e12 if fwd_launch_ms > 0 else float("nan")
    # DRAM bytes of one backward pair launch from the committed ncu --set full capture (profiles/ncu_traffic.json:
    # the full (i > j) chunk pair at this launch shape; the diagonal pairs move about half)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("attn_bwd_kernel_bytes_per_launch")

    # ---------------------------------------------------------------- end to end (host buffers)
    # The step through the library's host-memory calls (include/fpdt.h fpdt_attn_fwd_host / fpdt_attn_bwd_host): q, k,
    # v, dO live in pinned host memory and o, dq, dk, dv are written back to pinned host memory, every step, inside
    # the timed region.  The library moves the caller's rows chunk by chunk inside its own copy schedule (chunk m's
    # upload just ahead of its first reader, each chunk's outputs as soon as they are final); at world size 1 q_i and
    # dO_i reach the GPU through the chunk fetches themselves.
    e2e = None
    if not args.no_e2e:
        hin = [torch.empty(t.shape, dtype=bf, pin_memory=True) for t in (q, k, v, do)]
        for h_, t in zip(hin, (q, k, v, do)):
            h_.copy_(t)
        hq, hk, hv, hdo = hin
        hout = [torch.empty(t.shape, dtype=bf, pin_memory=True) for t in (o, dq, dk, dv)]
        ho, hdq, hdk, hdv = hout
        h2d_b = sum(t.numel() * 2 for t in hin)
        d2h_b = sum(t.numel() * 2 for t in hout)

        def host_step():
            fpdt.fpdt_attn_fwd_host(ctx, hq, hk, hv, ho, None, s_local, Hq, Hkv, d, 1, C, world, fpdt.FPDT_BF16,
                                    offload, 0.0, stream)
            fpdt.fpdt_attn_bwd_host(ctx, ho, hdo, hdq, hdk, hdv, s_local, Hq, Hkv, d, 1, C, world, fpdt.FPDT_BF16,
                                    offload, 0.0, stream)

        def run_e2e(n_steps):
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(n_steps):
                host_step()
            end.record(stream)
            torch.cuda.synchronize()
            return start.elapsed_time(end)

        run_e2e(2)  # warm-up (the library's device mirrors of the caller's tensors)
        barrier()
        sio0 = ctx.stats()
        e2e_ms = max_over_ranks(run_e2e(args.steps) / args.steps)
        sio1 = ctx.stats()
        barrier()
        # parity of the timed path: the host outputs equal the device-memory step's (same inputs, same kernels)
        same = bool(torch.equal(ho.to(o.device), o) and torch.equal(hdk.to(dk.device), dk)
                    and torch.equal(hdv.to(dv.device), dv))
        e2e = {"value": S / (e2e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "io_bytes_counted_per_step": {
                   "h2d": (sio1["bytes_io_h2d"] - sio0["bytes_io_h2d"]) // args.steps,
                   "d2h": (sio1["bytes_io_d2h"] - sio0["bytes_io_d2h"]) // args.steps},
               "outputs_equal_device_path": same,
               "path": "pinned host q,k,v,dO -> fpdt_attn_fwd_host + fpdt_attn_bwd_host (C-ABI, host pointers) -> "
                       "pinned host o,dq,dk,dv; the library stages the rows per chunk on its copy streams "
                       "(world size 1: dO_i and q_i reach the GPU through the chunk fetches, counted in pcie bytes)"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        dt, fl = oracle_sample(S_sample=8192)
        cpu = {"value": projected_tokens_per_s(dt, fl, S, Hq, d), "unit": "tokens/s", "cores": cpu_cores(),
               "kind": "oracle", "seconds": dt,
               "sample": "fp64 numpy oracle (oracle/attention.py) fwd+bwd of the first 8192 tokens x 2 heads "
                         "(d=80); tokens/s projected to the full workload by algorithmic FLOPs"}

    line = {
        "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded counter-based generator, normal)",
        "tflops_per_gpu": tflops_gpu,
        "frac_of_peak": tflops_gpu / sustained,
        # MFU-style "model FLOPs": 12d per causal pair per q-head, no backward recompute of Q K^T
        "model_tflops_per_gpu": tflops_gpu * 12 / 14,
        "config": {"workload": W["name"], "S": S, "heads_q": Hq, "heads_kv": Hkv, "head_dim": d, "chunk": C,
                   "chunks": S // C, "s_local": s_local, "offload": offload, "causal": 1,
                   "parallelism": f"ulysses-sp{world}" + ("-nccl1" if world == 1 and args.exchange_path else ""), "l2": "inputs 2.7 GB/tensor >> 126 MB L2, no flush",
                   "flops_per_step": f_fwd + f_bwd, "flop_convention": "14*d per causal pair per q-head",
                   "sparsity": args.sparsity, "residency": args.residency or [0, 0],
                   "bwd_order": ["kv_outer", "q_outer"][st1["bwd_order"]]},
        "roofline": {"bound": "tensor", "kernel": "attn_bwd_pipe_kernel<80> (tcgen05 pair backward)",
                     "achieved": ach_bwd, "peak": sustained, "unit": "TFLOP/s", "frac": ach_bwd / sustained,
                     "traffic": traffic, "peak_source": peak_src + ", sustained bf16 (kernel timed inside a long step)",
                     "launch_ms": bwd_launch_ms, "launches_per_step": n_bwd // args.steps,
                     "fwd_kernel": {"achieved": ach_fwd, "frac": ach_fwd / sustained, "launch_ms": fwd_launch_ms,
                                    "launches_per_step": n_fwd // args.steps},
                     "kernel_share_of_step": (fwd_ms + bwd_ms) / args.steps / ms},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
        "pcie_bytes_per_step": {"h2d": h2d_lib, "d2h": d2h_lib},
        # offload / prefetch traffic of the library (per rank) against the host link: pinned copies measured on the
        # box at 55.6 GB/s H2D, 57.3 GB/s D2H (profiles/r01_box_probe.md); the transfers overlap compute
        "host_link": {"h2d_GBps": h2d_lib / (ms / 1e3) / 1e9, "d2h_GBps": d2h_lib / (ms / 1e3) / 1e9,
                      "measured_peak_GBps": {"h2d": 55.6, "d2h": 57.3}},
        "a2a_bytes_per_step": (st1["bytes_a2a"] - st0["bytes_a2a"]) // args.steps,
        # compute-stream accounting from the library's per-launch CUDA events: time the compute stream spent between
        # consecutive pair kernels of one call (waiting for an exchange, a fetch or a support kernel), and the step
        # time not covered by pair kernels at all (that plus the fwd/bwd preambles, D preprocess and converts)
        "compute_stream": {"pair_kernel_ms_per_step": (fwd_ms + bwd_ms) / args.steps,
                           "gap_ms_per_step": gap_ms / args.steps, "gaps_per_step": n_gaps // args.steps,
                           "exposed_ms_per_step": ms - (fwd_ms + bwd_ms) / args.steps},
        "max_seq_per_gpu": max_seq_record(),
        # the all-to-alls on the comm stream (p > 1): CUDA events around each exchange; bus GB/s = bytes sent to other
        # ranks / exchange time (NVLink 5: 900 GB/s per direction per GPU)
        "exchange": None if (world == 1 and not args.exchange_path) else {
            "ms_per_step": xch["total_ms"] / args.steps, "count_per_step": xch["n"] // args.steps,
            "bytes_per_step": xch["bytes"] // args.steps,
            "bus_GBps": (xch["bytes"] / (xch["total_ms"] / 1e3) / 1e9) if xch["total_ms"] > 0 else None,
            "first_ms": xch["first_ms"], "last_ms": xch["last_ms"]},
        "device_bytes_library": st1["device_bytes"],
        "wall_s_timed": wall,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--offload", type=int, default=1)
    ap.add_argument("--seq", type=int, default=0, help="override S (testing)")
    ap.add_argument("--chunk", type=int, default=0, help="override the chunk size (testing)")
    ap.add_argument("--sparsity", type=float, default=0.0,
                    help="block sparsity rho (PAPER.md §5.6 / Table sparsity): fraction of causal chunk blocks dropped")
    ap.add_argument("--residency", type=int, nargs=2, default=None, metavar=("KV_CHUNKS", "Q_CHUNKS"),
                    help="HBM residency budget (fpdt_set_residency): first KV chunks / last query-side chunks kept on "
                         "the device")
    ap.add_argument("--bwd-order", default="kv", choices=["kv", "q", "auto"],
                    help="backward loop order (fpdt_set_bwd_order): kv = the paper's (KV outer), q = GQA-aware Q outer")
    ap.add_argument("--exchange-path", action="store_true",
                    help="N = 1: run the sequence-parallel schedule through a one-rank NCCL communicator (pack, "
                         "ncclAlltoAll, unpack per chunk) instead of the in-place world-size-1 path")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="A/B check: time the step without the library's per-launch CUDA events (no roofline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
