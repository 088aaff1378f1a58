"""CTA-pair MMA micro-benchmark (include/fpdt_diag.h fpdt_selftest_pair): SM cycles per SS MMA for the single-CTA
M = 128 form and the CTA-pair M = 256 form (cta_group::2) at several N, all 148 SMs busy.  The pair form does twice
the work of one M = 128 MMA per issue; per SM it reads its own 128 x 16 A slice and half of B."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_16978_b200 import fpdt  # noqa: E402

out = torch.zeros(1, device="cuda")
lib = fpdt.diag()
res = []
for mode in (0, 1, 2):
    for n in (64, 80, 96, 128, 160, 192, 256):
        if mode == 0 and n > 256:
            continue
        vals = []
        for _ in range(3):
            rc = lib.fpdt_selftest_pair(mode, n, 4096, fpdt.c_void_p(out.data_ptr()), None)
            assert rc == 0, rc
            torch.cuda.synchronize()
            vals.append(float(out.item()))
        clk = sorted(vals)[1]
        M = 256 if mode == 1 else 128
        # FLOP per busy SM per clock: an M x N x 16 MMA is 2*M*N*16 FLOP, spread over 1 (modes 0, 2) or 2 (mode 1) SMs
        fpc = 2 * M * n * 16 / clk / (2 if mode == 1 else 1)
        res.append({"mode": ["cta_group::1 M=128", "cta_group::2 M=256", "cta_group::1 M=128, partner SM idle"][mode],
                    "N": n, "clk_per_mma": clk,
                    "flop_per_clk_per_sm": fpc})
        print(json.dumps(res[-1]), flush=True)
