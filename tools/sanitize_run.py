#!/usr/bin/env python
"""One fwd + bwd at BASELINE.json configs[0]'s shape (S = 4096, 8 heads, d = 64, C = 1024; fp32 and bf16, world size 1
and a p = 2 in-process group), for compute-sanitizer (memcheck / racecheck / synccheck; tools/gpu_sanitizer.sh).
Checks nothing itself beyond finiteness: the sanitizer's report is the result."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from fpdt_testlib import inputs, run_cuda  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
S, H, d, C = 4096, 8, 64, 1024
x = inputs("normal", 0, S, H, H, d)
if which in ("all", "fp32"):
    r = run_cuda(x, C, "fp32", 1)
    assert all(np.isfinite(r[n]).all() for n in ("o", "lse", "dq", "dk", "dv"))
    print("fp32 p=1 ok", flush=True)
if which in ("all", "bf16"):
    r = run_cuda(x, C, "bf16", 1)
    assert all(np.isfinite(r[n]).all() for n in ("o", "lse", "dq", "dk", "dv"))
    print("bf16 p=1 ok", flush=True)
if which in ("all", "p2"):
    from test_gpu_multirank import run_group
    r = run_group(x, 2, C, "bf16", 1)
    assert all(np.isfinite(r[n]).all() for n in ("o", "lse", "dq", "dk", "dv"))
    print("bf16 p=2 ok", flush=True)
