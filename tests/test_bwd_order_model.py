"""Host-side model of the backward loop orders (include/fpdt.h fpdt_bwd_host_bytes, the numbers FPDT_BWD_AUTO
compares) against an independent count of each schedule (tests/fpdt_testlib.expected_bwd_bytes, written from
PAPER.md L365 for the KV-outer order and from SURVEY §8(f) NEXT-1 for the Q-outer one).  Host-only: no GPU."""
import numpy as np
import pytest

import fpdt_inputs as gen
from fpdt_testlib import expected_bwd_bytes


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("p,Hq,Hkv,d,eb", [(1, 32, 32, 80, 2), (4, 32, 8, 128, 2), (8, 64, 8, 128, 2),
                                            (2, 8, 2, 64, 4)])
@pytest.mark.parametrize("res", [(0, 0), (2, 3), (9, 9)])
@pytest.mark.parametrize("rho", [0.0, 0.4])
def test_model_matches_schedule_count(order, p, Hq, Hkv, d, eb, res, rho):
    from paper_2408_16978_b200 import fpdt
    C, u = 1024 * p, 8
    s_local = u * C // p
    keep = gen.sparsity_plan(u, rho, seed=3) if rho else None
    got = fpdt.fpdt_bwd_host_bytes(order, s_local, Hq, Hkv, d, C, p, 0 if eb == 2 else 1, res[0], res[1], keep)
    h2d, d2h = expected_bwd_bytes(order, u, C, Hq // p, Hkv // p, d, eb, keep=keep, rkv=min(res[0], u),
                                  rq=min(res[1], u))
    assert got == h2d + d2h


def test_model_gqa_prefers_q_outer_and_mha_kv_outer():
    """The survey's claim: with G = 4..8 the Q-outer order moves several times fewer host bytes
    per pair; for MHA the paper's order moves fewer."""
    from paper_2408_16978_b200 import fpdt
    K = 65536
    c3 = [fpdt.fpdt_bwd_host_bytes(o, 2 * 1024 * 1024 // 4, 32, 8, 128, K, 4, 0) for o in (0, 1)]
    c5 = [fpdt.fpdt_bwd_host_bytes(o, 1024 * 1024 // 8, 64, 8, 128, K, 8, 0) for o in (0, 1)]
    c2 = [fpdt.fpdt_bwd_host_bytes(o, 512 * 1024, 32, 32, 80, K, 1, 0) for o in (0, 1)]
    assert c3[0] / c3[1] > 2 and c5[0] / c5[1] > 3 and c2[1] > c2[0]


def test_model_errors():
    from paper_2408_16978_b200 import fpdt
    with pytest.raises(fpdt.FpdtError):
        fpdt.fpdt_bwd_host_bytes(2, 4096, 4, 4, 64, 1024, 1, 0)          # AUTO is not a schedule
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_bwd_host_bytes(0, 4000, 4, 4, 64, 1024, 1, 0)          # S % C != 0
    assert e.value.code == fpdt.FPDT_ERR_DIVISIBILITY
    with pytest.raises(fpdt.FpdtError):
        fpdt.fpdt_bwd_host_bytes(0, 4096, 4, 4, 64, 1024, 1, 0, keep=np.ones((3, 3), bool))


@pytest.mark.parametrize("args,code", [
    ((0, 0, 4, 4, 64, 1024, 1, 0), "FPDT_ERR_ARG"),            # empty shard
    ((0, 4096, 0, 4, 64, 1024, 1, 0), "FPDT_ERR_ARG"),         # no heads
    ((0, 4096, 4, 4, 96, 1024, 1, 0), "FPDT_ERR_UNSUPPORTED"),  # head_dim without a kernel
    ((0, 4096, 4, 4, 64, 1024, 1, 7), "FPDT_ERR_UNSUPPORTED"),  # dtype
    ((0, 4096, 4, 4, 64, 1000, 1, 0), "FPDT_ERR_DIVISIBILITY"),  # C % 256
    ((0, 4096, 4, 4, 64, 1024, 3, 0), "FPDT_ERR_DIVISIBILITY"),  # C % p
    ((0, 4096, 6, 4, 64, 1024, 1, 0), "FPDT_ERR_DIVISIBILITY"),  # Hq % Hkv
    ((0, 4096, 4, 2, 64, 1024, 4, 0), "FPDT_ERR_DIVISIBILITY"),  # Hkv % p
])
def test_shape_validation_host_only(args, code):
    """The divisibility / support rules of include/fpdt.h on the host path every call shares."""
    from paper_2408_16978_b200 import fpdt
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_bwd_host_bytes(*args)
    assert e.value.code == getattr(fpdt, code)


def test_single_chunk_degenerate():
    """u = 1: the backward is one diagonal pair in either order and moves nothing through the host but kv_0 and
    q_0, dO_0 once each."""
    from paper_2408_16978_b200 import fpdt
    C, Hq, Hkv, d = 1024, 4, 2, 64
    for order in (0, 1):
        got = fpdt.fpdt_bwd_host_bytes(order, C, Hq, Hkv, d, C, 1, 0)
        assert got == C * 2 * Hkv * d * 2 + 2 * C * Hq * d * 2
