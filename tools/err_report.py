"""Print the normwise max relative error of every output against the fp64 oracle for a few input distributions at
one head shape (bf16, offload on).  A/B helper for kernel-precision changes: python tools/err_report.py [d] [S] [C]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from fpdt_testlib import inputs, oracle_full, rel_err, run_cuda  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 80
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
C = int(sys.argv[3]) if len(sys.argv) > 3 else 512
for dist in ("normal", "peaky", "drift", "drift32", "extreme", "sink", "class"):
    x = inputs(dist, 3, S, 2, 2, d)
    res = run_cuda(x, C, "bf16", 1)
    ref = oracle_full(x)
    print(json.dumps({"d": d, "dist": dist, **{n: float("%.3g" % rel_err(res[n], ref[n]))
                                              for n in ("o", "lse", "dq", "dk", "dv")}}), flush=True)
