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
