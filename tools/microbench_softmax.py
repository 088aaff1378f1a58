"""Throughput of the forward softmax's exponential stage in isolation (fpdt_selftest_softmax)."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_16978_b200 import _lib

lib = _lib.load_diag()
out = torch.zeros(4, device="cuda")
for what, cols, thr_list in ((0, 128, (128, 256)), (1, 64, (128, 256, 512))):
    for every, name in ((4, "25% poly"), (0, "all MUFU"), (2, "50% poly"), (8, "12% poly")):
        for thr in thr_list:
            for iters in (4, 64):
                assert lib.fpdt_selftest_softmax(what, thr, every, iters, ctypes.c_void_p(out.data_ptr()), None) == 0
                torch.cuda.synchronize()
            c = out[0].item()
            print(f"{cols:3d} cols {name:9s} {thr:4d} thr/SM ({thr // 128} warp/SMSP): {c:7.1f} clk/row -> "
                  f"{thr * cols / c / 4:.2f} elem/clk/SMSP")
