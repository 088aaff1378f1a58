#!/usr/bin/env python
"""Where the end-to-end gap comes from (bench.py's e2e vs the device-timed step): the bench workload's step loop with
the host copies of its inputs (q, k, v, dO: pinned host -> device) and outputs (o, dq, dk, dv: device -> pinned host)
switched on separately.  Same double-buffered copy stream as bench.py.  One JSON line per variant.

    python tools/e2e_probe.py [--steps 3] [--seq 524288]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fpdt_inputs as gen  # noqa: E402
from paper_2408_16978_b200 import _lib, fpdt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--one-set", action="store_true", help="one buffer set for every step (as bench.py's device loop)")
    ap.add_argument("--variants", nargs="+", default=["none", "uploads", "downloads", "both", "none_again"])
    ap.add_argument("--warmup-copies", type=int, default=1, help="0: warm up without host copies")
    ap.add_argument("--no-pinned", action="store_true", help="do not allocate the pinned host buffers")
    a = ap.parse_args()
    S, H, d, C = a.seq, 32, 80, 65536
    genlib = _lib.load_generator()
    bf = torch.bfloat16

    def g(name):
        t = torch.empty(S, H, d, dtype=bf, device="cuda")
        assert genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name], 0, 0, S, H, d, S, 0, 1, C,
                                    ctypes.c_void_p(0)) == 0
        return t

    sets = []
    for _ in range(1 if a.one_set else 2):
        q, k, v, do = g("q"), g("k"), g("v"), g("do")
        sets.append(((q, k, v, do), tuple(torch.empty_like(t) for t in (q, q, k, v))))
    hin = [torch.empty(t.shape, dtype=bf, pin_memory=not a.no_pinned) for t in sets[0][0]]
    for h_, t in zip(hin, sets[0][0]):  # the uploads must carry the real inputs: the GPU's power draw (and so its
        h_.copy_(t)                      # power-capped clock) depends on the data -- zeros run at 1965 MHz, these at ~1600
    hout = [torch.empty(t.shape, dtype=bf, pin_memory=not a.no_pinned) for t in sets[0][1]]
    ctx = fpdt.FPDTContext()
    stream = torch.cuda.current_stream()
    cp = torch.cuda.Stream()

    def run(n, up, down):
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cp.wait_event(e0)

        def upload(i):
            b = i % 2
            with torch.cuda.stream(cp):
                if i >= 2:
                    cp.wait_event(ev_done[b])
                if up:
                    for h_, t in zip(hin, sets[b][0]):
                        t.copy_(h_, non_blocking=True)
                ev_in[b].record(cp)

        upload(0)
        if n > 1:
            upload(1)
        for i in range(n):
            b = i % 2
            (qi, ki, vi, doi), (oi, dqi, dki, dvi) = sets[b]
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[b])
            fpdt.fpdt_attn_fwd(ctx, qi, ki, vi, oi, None, S, H, H, d, 1, C, 1, fpdt.FPDT_BF16, 1, 0.0, stream)
            fpdt.fpdt_attn_bwd(ctx, oi, doi, dqi, dki, dvi, S, H, H, d, 1, C, 1, fpdt.FPDT_BF16, 1, 0.0, stream)
            ev_done[b].record(stream)
            with torch.cuda.stream(cp):
                cp.wait_event(ev_done[b])
                if down:
                    for h_, t in zip(hout, sets[b][1]):
                        h_.copy_(t, non_blocking=True)
                ev_out[b].record(cp)
            if i + 2 < n:
                upload(i + 2)
        stream.wait_event(ev_out[(n - 1) % 2])
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    from bench import ClockSampler
    if a.one_set:
        sets.append(sets[0])
    run(2, bool(a.warmup_copies), bool(a.warmup_copies))
    table = {"none": (False, False), "uploads": (True, False), "downloads": (False, True), "both": (True, True),
             "none_again": (False, False)}
    for name in a.variants:
        up, down = table[name]
        cs = ClockSampler(torch.cuda.current_device())
        cs.start()
        ms = run(a.steps, up, down)
        clocks = cs.stop()
        print(json.dumps({"tool": "e2e_probe", "variant": name, "one_set": a.one_set, "steps": a.steps, "ms_per_step": ms,
                          "tokens_per_s": S / (ms / 1e3), "clocks": clocks}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
