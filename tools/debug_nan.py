"""d = 64 forward, extreme logits: the diagonal pair kernel alone (debug aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import fpdt_inputs as gen
from paper_2408_16978_b200 import fpdt

lib = fpdt.diag()
x = gen.make_inputs("extreme", 61, 2048, 4, 2, 64)
for d, lo, n in ((64, 1536, 512), (80, 1536, 512)):
    x = gen.make_inputs("extreme", 61, 2048, 4, 2, d)
    q, k, v = (torch.tensor(x[m][lo:lo + n]).to(torch.bfloat16).cuda().contiguous() for m in ("q", "k", "v"))
    o = torch.empty_like(q)
    lse = torch.empty(4, n, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    assert lib.fpdt_debug_pair(0, d, 1, P(q), P(k), P(v), None, None, None, P(o), P(lse), None, n, 4, 2, None, 0, None) == 0
    torch.cuda.synchronize()
    qq = x["q"][lo:lo + n, 2].astype(np.float64)
    kk = x["k"][lo:lo + n, 1].astype(np.float64)
    s = qq @ kk.T / np.sqrt(d) * np.log2(np.e)
    for r in range(4):
        ref = np.logaddexp2.reduce(s[r, :r + 1])
        print(f"d={d} row {r} head 2: lse2 gpu {lse[2, r].item():.4f} ref {ref:.4f}; o[0:3] {o[r, 2, :3].float().tolist()}")
