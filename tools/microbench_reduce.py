"""dQ reduce-add path throughput (fpdt_selftest_reduce): SM cycles and bytes/clk/SM per 40 KB tile."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_16978_b200 import _lib

lib = _lib.load_diag()
g = torch.zeros(2 * 148 * 10240 + 1024, device="cuda")
out = torch.zeros(4, device="cuda")
names = {0: "3 swizzled boxes", 1: "1-D bulk 40KB", 2: "10 x 4KB bulk", 3: "1 box [128x80]", 4: "bulk STORE 40KB",
         5: "boxes + 40KB load", 6: "40KB load only"}
for mode in (0, 5, 6, 1, 4):
    for inflight in (1, 2):
        for shared in (0, 1):
            for iters in (8, 128):
                rc = lib.fpdt_selftest_reduce(mode, iters, inflight, shared, ctypes.c_void_p(g.data_ptr()),
                                              ctypes.c_void_p(out.data_ptr()), None)
                assert rc == 0, rc
                torch.cuda.synchronize()
            c = out[0].item()
            print(f"{names[mode]:18s} inflight={inflight} shared={shared}: {c:7.0f} clk/tile -> {40960 / c:5.1f} B/clk/SM")
