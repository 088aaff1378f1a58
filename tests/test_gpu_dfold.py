"""The backward's D fold (d = 80: dP^T = V dO^T - D as a sixth k-step, with D entering as a bf16 hi / lo pair; DESIGN.md
§6) where it is most exposed:
  * "flat values": v_j = v + 0.01 noise, so dP_ij = <dO_i, v_j> is within ~1% of D_i = <dO_i, O_i> and
    dS_ij = P_ij (dP_ij - D_i) is a small difference of large terms -- the hi / lo split carries D to ~2^-16
    relative, two orders below the bf16 rounding of dS itself;
  * dO scaled by 1e3 and by 1e-3 (D and every gradient scale with it; the hi / lo pair must not under- or
    overflow).
Each against the fp64 oracle on the same bf16-rounded inputs (normwise max relative error <= 1e-2)."""
import numpy as np
import pytest
import torch

from fpdt_testlib import TOL, inputs, oracle_full, rel_err, run_cuda

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.tensor(a).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("case", ["flat_v", "do_x1e3", "do_x1e-3"])
@pytest.mark.parametrize("Hq,Hkv", [(2, 2), (4, 1)])
def test_dfold_exposed_cases(case, Hq, Hkv):
    S, d, C = 2048, 80, 512
    x = dict(inputs("normal", 11, S, Hq, Hkv, d))
    if case == "flat_v":
        rng = np.random.default_rng(5)
        v0 = rng.standard_normal((1, Hkv, d))
        x["v"] = _bf16(v0 + 0.01 * x["v"])
    elif case == "do_x1e3":
        x["do"] = _bf16(x["do"] * 1e3)
    else:
        x["do"] = _bf16(x["do"] * 1e-3)
    got = run_cuda(x, C, "bf16", 1)
    ref = oracle_full(x)
    errs = {n: rel_err(got[n], ref[n]) for n in ("o", "lse", "dq", "dk", "dv")}
    assert all(np.isfinite(got[n]).all() for n in ("o", "lse", "dq", "dk", "dv"))
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
