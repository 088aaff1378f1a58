"""Key/value fetch strategies of the offloaded schedule (fpdt_set_fetch_strategy; PAPER.md
L311-323): A = every rank fetches its own chunks over its own host link, B = rank 0 keeps every rank's key/value chunks,
fetches all p blocks and scatters them (gather at the offload).  On one GPU through the in-process group (p = 2, 4):
B must give bitwise the same O, lse, dK, dV as A (the same kernels read the same bytes), dQ within the reduce-order
bound, oracle parity, and the host-link bytes must move from ranks r > 0 to rank 0 exactly as the schedule says."""
import numpy as np
import pytest

import fpdt_inputs as gen
from fpdt_testlib import TOL, oracle_full, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,Hq,Hkv,d", [(2, 4, 2, 80), (4, 8, 4, 128)])
def test_leader_fetch_matches_per_rank(p, Hq, Hkv, d):
    from paper_2408_16978_b200 import fpdt
    from test_gpu_multirank import run_group
    S, C = 2048, 512  # u = 4
    u = S // C
    x = gen.make_inputs("drift", 81, S, Hq, Hkv, d)
    st_a, st_b = {}, {}
    a = run_group(x, p, C, "bf16", 1, stats=st_a, fetch=fpdt.FPDT_FETCH_PER_RANK, debug_checks=True)
    b = run_group(x, p, C, "bf16", 1, stats=st_b, fetch=fpdt.FPDT_FETCH_LEADER, debug_checks=True)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(a[n], b[n]), n
    assert rel_err(b["dq"], a["dq"]) < 2.0 ** -8
    errs = {n: rel_err(b[n], r) for n, r in oracle_full(x).items()}
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
    # host-link bytes: the key/value fetches (forward: one per earlier chunk of every chunk; backward: one per key
    # chunk) move from every rank's link to rank 0's
    blk = C * 2 * (Hkv // p) * d * 2
    n_fetch = u * (u - 1) // 2 + u
    assert st_b[0]["bytes_h2d"] - st_a[0]["bytes_h2d"] == n_fetch * (p - 1) * blk
    for r in range(1, p):
        assert st_a[r]["bytes_h2d"] - st_b[r]["bytes_h2d"] == n_fetch * blk
    # the offloads move the same way (rank 0 writes every rank's key/value chunk)
    assert st_b[0]["bytes_d2h"] - st_a[0]["bytes_d2h"] == u * (p - 1) * blk
    for r in range(1, p):
        assert st_a[r]["bytes_d2h"] - st_b[r]["bytes_d2h"] == u * blk


def test_leader_fetch_with_sparsity_and_residency():
    from paper_2408_16978_b200 import fpdt
    from test_gpu_multirank import run_group
    S, Hq, Hkv, d, C, p = 2048, 4, 2, 64, 256, 2  # u = 8
    keep = gen.sparsity_plan(S // C, 0.3, seed=3)
    x = gen.make_inputs("normal", 82, S, Hq, Hkv, d)
    a = run_group(x, p, C, "bf16", 1, keep=keep, residency=(2, 2), fetch=fpdt.FPDT_FETCH_PER_RANK)
    b = run_group(x, p, C, "bf16", 1, keep=keep, residency=(2, 2), fetch=fpdt.FPDT_FETCH_LEADER)
    for n in ("o", "lse", "dk", "dv"):
        assert np.array_equal(a[n], b[n]), n
