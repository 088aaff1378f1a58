"""Error behaviour of the C-ABI (include/fpdt.h status codes), on the GPU."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _t(S, H, d, dt=torch.bfloat16):
    return torch.zeros(S, H, d, dtype=dt, device="cuda")


def test_status_codes():
    from paper_2408_16978_b200 import fpdt
    ctx = fpdt.FPDTContext()
    q, k, v, o = _t(1024, 2, 64), _t(1024, 2, 64), _t(1024, 2, 64), _t(1024, 2, 64)
    with pytest.raises(fpdt.FpdtError) as e:      # backward before forward
        fpdt.fpdt_attn_bwd(ctx, o, o, q, k, v, 1024, 2, 2, 64, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_STATE
    with pytest.raises(fpdt.FpdtError) as e:      # unsupported head_dim
        fpdt.fpdt_attn_fwd(ctx, _t(1024, 2, 96), _t(1024, 2, 96), _t(1024, 2, 96), _t(1024, 2, 96), None,
                           1024, 2, 2, 96, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_UNSUPPORTED
    with pytest.raises(fpdt.FpdtError) as e:      # chunk not a multiple of 256
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, 1024, 2, 2, 64, 1, 384, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_DIVISIBILITY
    with pytest.raises(fpdt.FpdtError) as e:      # S % C != 0
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, 1024, 2, 2, 64, 1, 768, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_DIVISIBILITY
    with pytest.raises(fpdt.FpdtError) as e:      # GQA group must divide
        fpdt.fpdt_attn_fwd(ctx, _t(1024, 3, 64), _t(1024, 2, 64), _t(1024, 2, 64), _t(1024, 3, 64), None,
                           1024, 3, 2, 64, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_DIVISIBILITY
    with pytest.raises(fpdt.FpdtError) as e:      # empty sequence
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, 0, 2, 2, 64, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_ARG
    with pytest.raises(fpdt.FpdtError) as e:      # empty sequence, host-memory form
        fpdt.fpdt_attn_fwd_host(ctx, q.cpu(), k.cpu(), v.cpu(), o.cpu(), None, 0, 2, 2, 64, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_ARG
    with pytest.raises(fpdt.FpdtError) as e:      # null pointer
        fpdt.fpdt_attn_fwd(ctx, None, k, v, o, None, 1024, 2, 2, 64, 1, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_ARG
    with pytest.raises(fpdt.FpdtError) as e:      # non-causal not supported
        fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, 1024, 2, 2, 64, 0, 256, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_UNSUPPORTED
    fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, 1024, 2, 2, 64, 1, 256, 1, 0, 1)
    with pytest.raises(fpdt.FpdtError) as e:      # backward with different arguments than the forward
        fpdt.fpdt_attn_bwd(ctx, o, o, q, k, v, 1024, 2, 2, 64, 1, 512, 1, 0, 1)
    assert e.value.code == fpdt.FPDT_ERR_STATE
    ctx.close()


def test_host_arena_exhaustion():
    """A pinned host store that cannot be allocated is FPDT_ERR_HOST_OOM (SURVEY §4 tier 7), and the failed create
    leaves the device usable."""
    from paper_2408_16978_b200 import fpdt
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.FPDTContext(host_arena_bytes=1 << 50)   # 1 PiB of pinned memory
    assert e.value.code == fpdt.FPDT_ERR_HOST_OOM
    ctx = fpdt.FPDTContext()
    ctx.close()


def test_device_working_set_exhaustion():
    """A working set the device cannot hold is FPDT_ERR_DEVICE_OOM before any kernel runs (the saved lse of a
    2^40-token sequence alone is 4 TiB), and the context stays usable."""
    from paper_2408_16978_b200 import fpdt
    q = _t(256, 1, 64)
    o = torch.empty_like(q)
    ctx = fpdt.FPDTContext()
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.fpdt_attn_fwd(ctx, q, q, q, o, None, 1 << 40, 1, 1, 64, 1, 1 << 20, 1, fpdt.FPDT_BF16, 1)
    assert e.value.code == fpdt.FPDT_ERR_DEVICE_OOM
    with pytest.raises(fpdt.FpdtError) as e:   # no forward was saved
        fpdt.fpdt_attn_bwd(ctx, o, o, q, q, q, 1 << 40, 1, 1, 64, 1, 1 << 20, 1, fpdt.FPDT_BF16, 1)
    assert e.value.code == fpdt.FPDT_ERR_STATE
    fpdt.fpdt_attn_fwd(ctx, q, q, q, o, None, 256, 1, 1, 64, 1, 256, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    ctx.close()


def test_nccl_init_times_out_instead_of_hanging(monkeypatch):
    """A rank whose peers never join: the non-blocking NCCL initialisation is bounded by FPDT_NCCL_TIMEOUT_S and
    fpdt_ctx_create returns FPDT_ERR_NCCL (SURVEY §5 failure detection)."""
    import time
    from paper_2408_16978_b200 import fpdt
    monkeypatch.setenv("FPDT_NCCL_TIMEOUT_S", "3")
    nid = fpdt.fpdt_get_unique_id()
    t0 = time.time()
    with pytest.raises(fpdt.FpdtError) as e:
        fpdt.FPDTContext(2, 0, nid)
    assert e.value.code == fpdt.FPDT_ERR_NCCL
    assert "timed out" in str(e.value)
    assert time.time() - t0 < 60


def test_debug_checks_catch_mismatched_ranks():
    """fpdt_set_debug_checks: ranks entering a collective call with different arguments get FPDT_ERR_ARG on every
    rank instead of mismatched all-to-alls; equal arguments pass (in-process group, p = 2)."""
    import threading
    from paper_2408_16978_b200 import fpdt
    S, H, d, C = 1024, 2, 64, 512
    group = fpdt.LocalGroup(2)
    codes = {}

    def rank_main(r, scale):
        torch.cuda.set_device(0)
        q, k, v, o = (_t(S // 2, H, d) for _ in range(4))
        ctx = fpdt.FPDTContext(2, r, group=group)
        ctx.set_debug_checks(True)
        try:
            fpdt.fpdt_attn_fwd(ctx, q, k, v, o, None, S // 2, H, H, d, 1, C, 2, 0, 1, scale)
            torch.cuda.synchronize()
            codes[r] = 0
        except fpdt.FpdtError as err:
            codes[r] = err.code
        ctx.close()

    for scales, want in (((0.0, 0.0), 0), ((0.0, 0.1), fpdt.FPDT_ERR_ARG)):
        th = [threading.Thread(target=rank_main, args=(r, scales[r])) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in th)
        assert codes == {0: want, 1: want}, codes
    group.close()
