"""Pins of oracle/block.py (the attention block with the fused QKV projection) against things
other than itself: central finite differences of L = <dO, O> in x and W (fp64, reading R21), and the special case
W = identity, where the block reduces to the pinned attention oracle on the columns of x (q heads, then k, then v:
the column convention of fpdt_block_fwd)."""
import numpy as np
import pytest

import fpdt_inputs as gen
from oracle import attention, block


def _loss(x, w, do, Hq, Hkv, d):
    o, _ = block.block_forward(x, w, Hq, Hkv, d)
    return float(np.sum(do * o))


@pytest.mark.parametrize("Hq,Hkv", [(2, 2), (4, 2)])
def test_block_gradients_finite_differences(Hq, Hkv):
    S, hidden, d = 8, 6, 4
    rng = np.random.default_rng(11)
    x = rng.standard_normal((S, hidden))
    w = rng.standard_normal((hidden, (Hq + 2 * Hkv) * d)) * 0.5
    do = rng.standard_normal((S, Hq, d))
    dx, dw = block.block_backward(x, w, do, Hq, Hkv, d)
    eps = 1e-5
    fd_x = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += eps
        xm[idx] -= eps
        fd_x[idx] = (_loss(xp, w, do, Hq, Hkv, d) - _loss(xm, w, do, Hq, Hkv, d)) / (2 * eps)
    fd_w = np.zeros_like(w)
    for idx in np.ndindex(*w.shape):
        wp, wm = w.copy(), w.copy()
        wp[idx] += eps
        wm[idx] -= eps
        fd_w[idx] = (_loss(x, wp, do, Hq, Hkv, d) - _loss(x, wm, do, Hq, Hkv, d)) / (2 * eps)
    assert np.abs(dx - fd_x).max() / np.abs(fd_x).max() < 1e-6
    assert np.abs(dw - fd_w).max() / np.abs(fd_w).max() < 1e-6


def test_block_identity_weight_reduces_to_attention():
    S, Hq, Hkv, d = 64, 4, 2, 8
    n = (Hq + 2 * Hkv) * d
    x = gen.make_inputs("normal", 3, S, Hq, Hkv, d)
    xs = np.concatenate([x["q"].reshape(S, -1), x["k"].reshape(S, -1), x["v"].reshape(S, -1)], axis=1)
    w = np.eye(n)
    o, lse = block.block_forward(xs, w, Hq, Hkv, d)
    ro, rlse = attention.attention_forward(x["q"], x["k"], x["v"])
    assert np.allclose(o, ro, rtol=0, atol=1e-13) and np.allclose(lse, rlse, rtol=0, atol=1e-13)
    dx, dw = block.block_backward(xs, w, x["do"], Hq, Hkv, d)
    dq, dk, dv = attention.attention_backward(x["q"], x["k"], x["v"], ro, rlse, x["do"])
    ref = np.concatenate([dq.reshape(S, -1), dk.reshape(S, -1), dv.reshape(S, -1)], axis=1)
    assert np.allclose(dx, ref, rtol=0, atol=1e-12)
    assert np.allclose(dw, xs.astype(np.float64).T @ ref, rtol=0, atol=1e-10)


def test_block_inputs_bf16_exact_and_scaled():
    x = gen.make_block_inputs("normal", 0, 256, 256, 4, 2, 32)
    for n in ("x", "w", "do"):
        assert np.array_equal(gen.bf16_round(x[n]), x[n]), n
    qkv = x["x"].astype(np.float64) @ x["w"]
    assert 0.7 < qkv.std() < 1.5


def test_bf16_rounding_helper():
    """The oracle's bf16 rounding (R27) against hand-worked bit patterns: ties to even, carries into the exponent,
    and the identity on bf16-representable values."""
    x = np.array([1.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 1.0 + 2.0 ** -7 + 2.0 ** -9, 2.0 - 2.0 ** -9, -3.5])
    want = np.array([1.0, 1.0, 1.0 + 2.0 ** -6, 1.0 + 2.0 ** -7, 2.0, -3.5])
    assert np.array_equal(block._bf16(x), want)


def test_bf16_intermediates_identity_weight():
    """With W = I and bf16 x, the projected q, k, v are already bf16: rounding them changes nothing in the forward;
    the backward then differs from the unrounded one only by the bf16 rounding of dq, dk, dv."""
    S, Hq, Hkv, d = 32, 2, 1, 8
    n = (Hq + 2 * Hkv) * d
    x = gen.make_inputs("normal", 5, S, Hq, Hkv, d)
    xs = np.concatenate([x["q"].reshape(S, -1), x["k"].reshape(S, -1), x["v"].reshape(S, -1)], axis=1)
    o1, l1 = block.block_forward(xs, np.eye(n), Hq, Hkv, d, bf16_intermediates=True)
    o0, l0 = block.block_forward(xs, np.eye(n), Hq, Hkv, d)
    assert np.array_equal(o1, o0) and np.array_equal(l1, l0)
    dx1, _ = block.block_backward(xs, np.eye(n), x["do"], Hq, Hkv, d, bf16_intermediates=True)
    dx0, _ = block.block_backward(xs, np.eye(n), x["do"], Hq, Hkv, d)
    assert np.array_equal(dx1, block._bf16(dx0))


def test_block_with_output_projection_finite_differences():
    """y = attention(x W) W_o: dx, dW, dW_o of L = <dY, y> against central finite differences."""
    S, hidden, d, Hq, Hkv = 8, 6, 4, 2, 1
    rng = np.random.default_rng(12)
    x = rng.standard_normal((S, hidden))
    w = rng.standard_normal((hidden, (Hq + 2 * Hkv) * d)) * 0.5
    wo = rng.standard_normal((Hq * d, hidden)) * 0.5
    dy = rng.standard_normal((S, hidden))

    def loss(x_, w_, wo_):
        o, _ = block.block_forward(x_, w_, Hq, Hkv, d)
        return float(np.sum(dy * block.output_forward(o, wo_)))

    o, _ = block.block_forward(x, w, Hq, Hkv, d)
    do, dwo = block.output_backward(o, wo, dy)
    dx, dw = block.block_backward(x, w, do, Hq, Hkv, d)
    eps = 1e-5
    for arr, grad, which in ((x, dx, 0), (w, dw, 1), (wo, dwo, 2)):
        fd = np.zeros_like(arr)
        for idx in np.ndindex(*arr.shape):
            ap, am = arr.copy(), arr.copy()
            ap[idx] += eps
            am[idx] -= eps
            args_p = [x, w, wo]
            args_m = [x, w, wo]
            args_p[which], args_m[which] = ap, am
            fd[idx] = (loss(*args_p) - loss(*args_m)) / (2 * eps)
        assert np.abs(grad - fd).max() / np.abs(fd).max() < 1e-6, which
