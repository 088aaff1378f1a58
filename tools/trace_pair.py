"""Time one chunk-pair kernel in isolation and print the warp-role timeline of one CTA
(fpdt_debug_pair).  Usage: python tools/trace_pair.py [fwd|bwd] [C] [heads] [d] [cta] [bwd kernel: 1 dispatch, 2 pipe,
3 CTA pair, 4 q64]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2408_16978_b200 import _lib

which = sys.argv[1] if len(sys.argv) > 1 else "bwd"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
H = int(sys.argv[3]) if len(sys.argv) > 3 else 32
d = int(sys.argv[4]) if len(sys.argv) > 4 else 80
cta = int(sys.argv[5]) if len(sys.argv) > 5 else 0
kern = int(sys.argv[6]) if len(sys.argv) > 6 else 1
causal = int(os.environ.get("CAUSAL", "1"))  # 0: a full (off-diagonal) pair
lib = _lib.load_diag()
torch.manual_seed(0)
bf = torch.bfloat16
q, k, v, do = (torch.randn(C, H, d, device="cuda").to(bf) for _ in range(4))
lse2 = torch.full((H, C), 12.0, device="cuda")
Dst = torch.zeros(H, C, device="cuda")
o = torch.empty_like(q)
lse = torch.empty(H, C, device="cuda")
dq = torch.zeros(C, H, d, device="cuda")
dk, dv = torch.empty_like(k), torch.empty_like(v)
trace = torch.zeros(16, 4096, dtype=torch.int64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None


def launch(tr):
    if which == "fwd":
        rc = lib.fpdt_debug_pair(0, d, causal, P(q), P(k), P(v), None, None, None, P(o), P(lse), None, C, H, H, tr, cta, None)
    else:
        rc = lib.fpdt_debug_pair(kern, d, causal, P(q), P(k), P(v), P(do), P(lse2), P(Dst), P(dq), P(dk), P(dv), C, H, H, tr,
                                 cta, None)
    assert rc == 0, rc


for _ in range(2):
    launch(None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    launch(None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = (4 if which == "fwd" else 10) * d * H * C * ((C + 1) / 2 if causal else C)
print(f"{which} {'pair' if causal else 'full pair'} C={C} H={H} d={d} kernel={kern}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
if len(sys.argv) > 7 and sys.argv[7] == "x":
    sys.exit(0)
launch(ctypes.c_void_p(trace.data_ptr()))
torch.cuda.synchronize()
t = trace.cpu().numpy()
names = {"bwd": ["sm:got_S", "sm:arr_P", "sm:got_dP", "sm:arr_dS", "mma:got_P", "mma:got_dS", "mma:iss_S+1",
                 "mma:got_dqempty", "mma:iss_dP+1", "dq:got_full", "sm:got_dsfree", "dq:reduce", "prod:got_qempty|sm:got_dsrx",
                 "sm:S_loaded", "sm:exp_done", "sm:dP_loaded|sm:stored"],
         "fwd": ["sm0:got_S", "sm0:arr_P", "sm1:got_S", "sm1:arr_P", "mma:got_P0", "mma:got_P1", "mma:got_K+1",
                 "prod:got_kvempty", "sm0:S_loaded", "sm0:max_done", "sm0:exp_done", "sm0:st_done",
                 "sm1:S_loaded", "sm1:max_done", "sm1:exp_done", "sm1:st_done"]}[which]
n = int((t[0][:1024] > 0).sum()) if which == "fwd" else int((t[0][:512] > 0).sum())
base = t[0][0]
print(f"traced CTA {cta}: {n} iterations; per-iteration deltas (SM clocks), iterations 4..{min(n, 12)}")
for i in range(4, min(n, 12)):
    row = [f"{nm}={(t[e][i] - base) if t[e][i] else -1:>9d}" for e, nm in enumerate(names)]
    print(f"it {i}: " + " ".join(row))
if n > 8:
    per = (t[0][n - 1] - t[0][4]) / (n - 5)
    print(f"mean clocks per iteration (sm got_S to got_S): {per:.0f}")
    for e, nm in enumerate(names):
        if e == 0:
            continue
        valid = [(t[e][i] - t[0][i]) for i in range(4, n - 1) if t[e][i] > 0]
        if valid:
            print(f"  {nm:>18s} - sm:got_S : median {np.median(valid):8.0f}")
if which == "fwd" and n > 8:
    # per-warp spread (events recorded by all four warps of a tile at slot 1024 * warp + iteration)
    for e, nm in ((10, "sm0:exp_done"), (1, "sm0:arr_P"), (14, "sm1:exp_done"), (3, "sm1:arr_P")):
        meds = []
        for w in range(4):
            valid = [(t[e][1024 * w + i] - t[0][i]) for i in range(4, min(n, 1024) - 1) if t[e][1024 * w + i] > 0]
            meds.append(f"{np.median(valid):7.0f}" if valid else "      -")
        print(f"  {nm:>14s} - sm:got_S per warp 0..3: " + " ".join(meds))
if which == "fwd" and n > 8:
    for e, sl, nm in ((6, 1024, "mma:S0(j+1) issued"), (6, 2048, "mma:S1(j+1) issued"), (4, 1024, "mma:PV0(j) issued"),
                      (5, 1024, "mma:PV1(j) issued")):
        valid = [(t[e][sl + i] - t[0][i]) for i in range(4, min(n, 1024) - 1) if t[e][sl + i] > 0]
        if valid:
            print(f"  {nm:>20s} - sm:got_S : median {np.median(valid):8.0f}")
if which == "bwd" and n > 8:
    for e, nm in ((14, "sm:exp_done"), (1, "sm:arr_P"), (3, "sm:arr_dS")):
        meds = []
        for w in range(8):
            valid = [(t[e][512 * w + i] - t[0][i]) for i in range(4, min(n, 512) - 1) if t[e][512 * w + i] > 0]
            meds.append(f"{np.median(valid):6.0f}" if valid else "     -")
        print(f"  {nm:>12s} - sm:got_S per warp 0..7: " + " ".join(meds))
