"""The all-to-all layout kernels (SURVEY §8(a) F3 pack, F10/B7 unpack, B2) against the sentinel index oracle of
oracle/layout.pack_index (SURVEY §4 tier 2; "exhaustive sentinel index oracle"), bitwise: every element
holds its own flat source index (fp32 for 4-byte elements, raw int16 bit patterns for 2-byte ones), so a packed
buffer must equal src.flat[pack_index] exactly, in the dense send layout, inside the combined q|k|v receive layout
(row stride and head offset) and from strided source rows (the fused-projection path); unpack inverts pack."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import layout

pytestmark = pytest.mark.gpu


def _relayout(which, src, dst, c, H, d, p, eb, peer_stride, row_ld, head0, seq_ld):
    from paper_2408_16978_b200 import fpdt
    rc = fpdt.diag().fpdt_debug_relayout(which, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), c, H,
                                        d, p, eb, peer_stride, row_ld, head0, seq_ld, None)
    assert rc == 0, rc
    torch.cuda.synchronize()


def _sentinel(n, eb):
    if eb == 4:
        return torch.arange(n, dtype=torch.float32, device="cuda")          # exact below 2^24
    return torch.arange(n, dtype=torch.int32, device="cuda").to(torch.int16)  # raw 16-bit patterns


@pytest.mark.parametrize("eb", [4, 2])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("d", [64, 80, 128])
def test_pack_matches_sentinel_oracle_and_unpack_inverts(p, d, eb):
    c, H = 32, 8
    n = c * H * d
    src = _sentinel(n, eb)
    hp = H // p
    packed = torch.empty_like(src)
    _relayout(0, src, packed, c, H, d, p, eb, c * hp * d, hp * d, 0, 0)
    want = src.cpu().numpy()[layout.pack_index(p, c, H, d)]
    assert np.array_equal(packed.cpu().numpy(), want)
    back = torch.empty_like(src)
    _relayout(1, packed, back, c, H, d, p, eb, c * hp * d, hp * d, 0, 0)
    assert torch.equal(back, src)


@pytest.mark.parametrize("p", [2, 4])
def test_pack_into_combined_buffer_from_strided_rows(p):
    """The forward's use: q, k, v rows of one chunk packed into ONE send buffer [p][c][hq + 2hkv][d] (k at head
    offset hq, v at hq + hkv), here from rows of a combined [c][Hq + 2Hkv][d] source (row stride Htot * d, the
    fused-projection path); the other heads of the destination are left untouched."""
    c, Hq, Hkv, d, eb = 32, 8, 4, 80, 4
    Htot = Hq + 2 * Hkv
    hq, hkv = Hq // p, Hkv // p
    hcomb = hq + 2 * hkv
    src = _sentinel(c * Htot * d, eb)                     # [c][Htot][d]
    dst = torch.full((p * c * hcomb * d,), -1.0, device="cuda")
    stride = c * hcomb * d
    for off, H, head0 in ((0, Hq, 0), (Hq, Hkv, hq), (Hq + Hkv, Hkv, hq + hkv)):
        sub = src[off * d:]                               # the q, k or v columns of each row
        _relayout(0, sub, dst, c, H, d, p, eb, stride, hcomb * d, head0, Htot * d)
    s = src.cpu().numpy().reshape(c, Htot, d)
    got = dst.cpu().numpy().reshape(p, c, hcomb, d)
    for peer in range(p):
        assert np.array_equal(got[peer, :, :hq], s[:, peer * hq:(peer + 1) * hq])
        assert np.array_equal(got[peer, :, hq:hq + hkv], s[:, Hq + peer * hkv:Hq + (peer + 1) * hkv])
        assert np.array_equal(got[peer, :, hq + hkv:], s[:, Hq + Hkv + peer * hkv:Hq + Hkv + (peer + 1) * hkv])
    # unpack each part back into strided rows of a fresh combined buffer
    out = torch.full_like(src, -1.0)
    for off, H, head0 in ((0, Hq, 0), (Hq, Hkv, hq), (Hq + Hkv, Hkv, hq + hkv)):
        _relayout(1, dst, out[off * d:], c, H, d, p, eb, stride, hcomb * d, head0, Htot * d)
    assert torch.equal(out, src)


def test_relayout_argument_errors():
    from paper_2408_16978_b200 import fpdt
    x = torch.zeros(1024, device="cuda")
    P = ctypes.c_void_p(x.data_ptr())
    lib = fpdt.diag()
    assert lib.fpdt_debug_relayout(2, P, P, 4, 4, 64, 1, 4, 1, 1, 0, 0, None) == fpdt.FPDT_ERR_ARG   # which
    assert lib.fpdt_debug_relayout(0, P, P, 4, 6, 64, 4, 4, 1, 1, 0, 0, None) == fpdt.FPDT_ERR_ARG   # H % p
    assert lib.fpdt_debug_relayout(0, P, P, 4, 4, 60, 1, 2, 1, 1, 0, 0, None) == fpdt.FPDT_ERR_ARG   # 16 B vectors
