"""Run the sm_100a unit micro-benchmarks in libfpdt.so (fpdt_selftest_perf) and print cycles/op."""
import ctypes
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_16978_b200 import _lib

lib = _lib.load_diag()
out = torch.zeros(4, device="cuda")
def run(what, n, iters):
    rc = lib.fpdt_selftest_perf(what, n, iters, ctypes.c_void_p(out.data_ptr()), None)
    torch.cuda.synchronize()
    assert rc == 0, rc
    return out[0].item()
for what, name in ((0, "SS mma"), (1, "TS mma")):
    for n in (16, 32, 64, 80, 128, 256):
        for chains in (1, 2):
            it = 2048 + chains if chains > 1 else 2048
            run(what, n, 64 + (chains if chains > 1 else 0))
            c = run(what, n, it)
            print(f"{name} M=128 N={n:3d} K=16 accum-chains={chains}: {c:7.2f} cyc/instr  ({128*n*16*2/c:7.0f} flop/cyc/SM)")
for what, name in ((2, "MUFU ex2"), (4, "poly exp2")):
    for thr in (128, 256, 512, 1024):
        run(what, thr, 64)
        c = run(what, thr, 4096)
        print(f"{name} {thr} thr/SM, 8 chains/thread: {c:.2f} cyc/op/thread -> {thr / c:.1f} ops/clk/SM")
run(3, 0, 64)
print(f"tcgen05.ld x32 per warp (4 warps, 4 in flight): {run(3, 0, 4096):.2f} cyc/op")
for what, name, per in ((5, "MUFU ex2 32 chains", 1), (7, "poly exp2 x2 16 pairs", 1), (8, "ex2.f16x2 16 chains", 2)):
    for thr in (128, 256, 512, 1024):
        run(what, thr, 64)
        c = run(what, thr, 4096)
        print(f"{name}: {thr} thr/SM: {c:.2f} cyc/elem/thread -> {per * thr / c:.1f} elem/clk/SM")
run(6, 128, 64)
print(f"MUFU ex2 latency (one dependent chain): {run(6, 128, 4096):.1f} cyc")
