"""Python binding of libfpdt (include/fpdt.h): argument marshalling only.

Every step of the FPDT attention path runs inside libfpdt.so (CUDA kernels for sm_100a, NCCL,
cudaMemcpyAsync); this module only turns torch tensors into device pointers and raises on a non-OK
status.  There is no fallback: a missing library raises ``FpdtLibraryMissing``.
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import c_float, c_int, c_int64, c_void_p

FPDT_OK, FPDT_ERR_ARG, FPDT_ERR_DIVISIBILITY, FPDT_ERR_UNSUPPORTED, FPDT_ERR_HOST_OOM, FPDT_ERR_DEVICE_OOM, \
    FPDT_ERR_STATE, FPDT_ERR_CUDA, FPDT_ERR_NCCL = range(9)
FPDT_BF16, FPDT_FP32 = 0, 1
FPDT_BWD_KV_OUTER, FPDT_BWD_Q_OUTER, FPDT_BWD_AUTO = 0, 1, 2
FPDT_FETCH_PER_RANK, FPDT_FETCH_LEADER = 0, 1
STATUS_NAMES = {0: "FPDT_OK", 1: "FPDT_ERR_ARG", 2: "FPDT_ERR_DIVISIBILITY", 3: "FPDT_ERR_UNSUPPORTED",
                4: "FPDT_ERR_HOST_OOM", 5: "FPDT_ERR_DEVICE_OOM", 6: "FPDT_ERR_STATE", 7: "FPDT_ERR_CUDA",
                8: "FPDT_ERR_NCCL"}

# names of every symbol include/fpdt.h declares (checked by the CPU tests against the built library)
EXPORTED = ("fpdt_get_unique_id", "fpdt_ctx_create", "fpdt_ctx_destroy", "fpdt_attn_fwd", "fpdt_attn_bwd",
            "fpdt_last_error", "fpdt_global_token", "fpdt_get_stats", "fpdt_set_kernel_timing", "fpdt_kernel_time",
            "fpdt_group_create", "fpdt_group_destroy", "fpdt_ctx_create_local", "fpdt_set_sparsity",
            "fpdt_set_residency", "fpdt_set_bwd_order", "fpdt_block_fwd", "fpdt_block_bwd", "fpdt_bwd_host_bytes",
            "fpdt_kernel_gaps", "fpdt_exchange_time", "fpdt_set_debug_checks", "fpdt_set_fetch_strategy",
            "fpdt_set_hidden_offload", "fpdt_attn_fwd_host", "fpdt_attn_bwd_host")
# include/fpdt_diag.h (libfpdt_diag.so: micro-benchmarks and direct kernel launches, not on the FPDT path)
DIAG_EXPORTED = ("fpdt_selftest_umma", "fpdt_selftest_perf", "fpdt_selftest_softmax", "fpdt_selftest_reduce",
                 "fpdt_selftest_pair", "fpdt_debug_relayout", "fpdt_debug_pair")


class FpdtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [("bytes_h2d", c_int64), ("bytes_d2h", c_int64), ("bytes_a2a", c_int64),
                ("kernel_launches", c_int64), ("attn_launches", c_int64), ("fetch_slots_highwater", c_int64),
                ("host_arena_bytes", c_int64), ("device_bytes", c_int64), ("bwd_order", c_int64),
                ("host_dkv_bytes", c_int64), ("stress_sleeps", c_int64), ("bytes_io_h2d", c_int64),
                ("bytes_io_d2h", c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _declare(lib):
    P = c_void_p
    lib.fpdt_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.fpdt_get_unique_id.restype = c_int
    lib.fpdt_ctx_create.argtypes = [c_int, c_int, ctypes.c_char_p, c_int, ctypes.c_size_t, ctypes.POINTER(P)]
    lib.fpdt_ctx_create.restype = c_int
    lib.fpdt_group_create.argtypes = [c_int, c_int, ctypes.POINTER(P)]
    lib.fpdt_group_create.restype = c_int
    lib.fpdt_group_destroy.argtypes = [P]
    lib.fpdt_group_destroy.restype = c_int
    lib.fpdt_ctx_create_local.argtypes = [P, c_int, c_int, ctypes.c_size_t, ctypes.POINTER(P)]
    lib.fpdt_ctx_create_local.restype = c_int
    lib.fpdt_ctx_destroy.argtypes = [P]
    lib.fpdt_ctx_destroy.restype = c_int
    lib.fpdt_attn_fwd.argtypes = [P, P, P, P, P, P, c_int64, c_int, c_int, c_int, c_int, c_int64, c_int, c_int, c_int,
                                  c_float, P]
    lib.fpdt_attn_fwd.restype = c_int
    lib.fpdt_attn_bwd.argtypes = [P, P, P, P, P, P, c_int64, c_int, c_int, c_int, c_int, c_int64, c_int, c_int, c_int,
                                  c_float, P]
    lib.fpdt_attn_bwd.restype = c_int
    for name in ("fpdt_attn_fwd_host", "fpdt_attn_bwd_host"):
        getattr(lib, name).argtypes = [P, P, P, P, P, P, c_int64, c_int, c_int, c_int, c_int, c_int64, c_int, c_int,
                                       c_int, c_float, P]
        getattr(lib, name).restype = c_int
    lib.fpdt_last_error.argtypes = []
    lib.fpdt_last_error.restype = ctypes.c_char_p
    lib.fpdt_global_token.argtypes = [c_int64, c_int64, c_int, c_int]
    lib.fpdt_global_token.restype = c_int64
    lib.fpdt_set_sparsity.argtypes = [P, P, c_int64]
    lib.fpdt_set_sparsity.restype = c_int
    lib.fpdt_set_residency.argtypes = [P, c_int64, c_int64]
    lib.fpdt_set_residency.restype = c_int
    lib.fpdt_block_fwd.argtypes = [P, P, P, P, P, P, P, c_int64, c_int, c_int, c_int, c_int, c_int, c_int64, c_int, c_int,
                                   c_int, c_float, P]
    lib.fpdt_block_fwd.restype = c_int
    lib.fpdt_block_bwd.argtypes = [P, P, P, P, P, P, P, P, P, c_int64, c_int, c_int, c_int, c_int, c_int, c_int64, c_int,
                                   c_int, c_int, c_float, P]
    lib.fpdt_block_bwd.restype = c_int
    lib.fpdt_bwd_host_bytes.argtypes = [c_int, c_int64, c_int, c_int, c_int, c_int64, c_int, c_int, c_int64, c_int64,
                                        P, c_int64, ctypes.POINTER(c_int64)]
    lib.fpdt_bwd_host_bytes.restype = c_int
    lib.fpdt_set_hidden_offload.argtypes = [P, c_int]
    lib.fpdt_set_hidden_offload.restype = c_int
    lib.fpdt_set_fetch_strategy.argtypes = [P, c_int]
    lib.fpdt_set_fetch_strategy.restype = c_int
    lib.fpdt_set_debug_checks.argtypes = [P, c_int]
    lib.fpdt_set_debug_checks.restype = c_int
    lib.fpdt_set_bwd_order.argtypes = [P, c_int]
    lib.fpdt_set_bwd_order.restype = c_int
    lib.fpdt_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
    lib.fpdt_get_stats.restype = c_int
    lib.fpdt_set_kernel_timing.argtypes = [P, c_int]
    lib.fpdt_set_kernel_timing.restype = c_int
    lib.fpdt_kernel_time.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int64),
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int64), c_int]
    lib.fpdt_kernel_time.restype = c_int
    lib.fpdt_kernel_gaps.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int64)]
    lib.fpdt_kernel_gaps.restype = c_int
    D_ = ctypes.POINTER(ctypes.c_double)
    lib.fpdt_exchange_time.argtypes = [P, D_, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), D_, D_]
    lib.fpdt_exchange_time.restype = c_int


def _declare_diag(lib):
    P = c_void_p
    lib.fpdt_selftest_umma.argtypes = [c_int, c_int, P, P, c_int, c_int, P, P]
    lib.fpdt_selftest_umma.restype = c_int
    lib.fpdt_selftest_reduce.argtypes = [c_int, c_int, c_int, c_int, P, P, P]
    lib.fpdt_selftest_reduce.restype = c_int
    lib.fpdt_selftest_softmax.argtypes = [c_int, c_int, c_int, c_int, P, P]
    lib.fpdt_selftest_softmax.restype = c_int
    lib.fpdt_debug_relayout.argtypes = [c_int, P, P, c_int64, c_int, c_int, c_int, c_int, c_int64, c_int64, c_int,
                                        c_int64, P]
    lib.fpdt_debug_relayout.restype = c_int
    lib.fpdt_selftest_pair.argtypes = [c_int, c_int, c_int, P, P]
    lib.fpdt_selftest_pair.restype = c_int
    lib.fpdt_selftest_perf.argtypes = [c_int, c_int, c_int, P, P]
    lib.fpdt_selftest_perf.restype = c_int
    lib.fpdt_debug_pair.argtypes = [c_int, c_int, c_int, P, P, P, P, P, P, P, P, P, c_int64, c_int, c_int, P, c_int, P]
    lib.fpdt_debug_pair.restype = c_int


def diag():
    """libfpdt_diag.so (include/fpdt_diag.h)."""
    return _lib.load_diag()


def lib():
    return _lib.load()


def _check(rc: int):
    if rc != FPDT_OK:
        raise FpdtError(rc, lib().fpdt_last_error().decode())


def _ptr(t):
    return None if t is None else c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def fpdt_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fpdt_get_unique_id(buf))
    return buf.raw


def fpdt_global_token(local_t: int, chunk_size: int, world_size: int, rank: int) -> int:
    return lib().fpdt_global_token(local_t, chunk_size, world_size, rank)


class LocalGroup:
    """fpdt_group: world_size ranks in this process on one device (single-GPU multi-rank tests)."""

    def __init__(self, world_size: int, device: int = 0):
        self.world_size = world_size
        h = c_void_p()
        _check(lib().fpdt_group_create(world_size, device, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            _check(lib().fpdt_group_destroy(self.handle))
            self.handle = None


class FPDTContext:
    """Owns one fpdt_ctx (NCCL comm or local group, streams, pinned host chunk store, device slots, saved
    state)."""

    def __init__(self, world_size: int = 1, rank: int = 0, nccl_id: bytes | None = None, device: int = 0,
                 host_arena_bytes: int = 0, group: LocalGroup | None = None):
        self.world_size, self.rank = world_size, rank
        h = c_void_p()
        if group is not None:
            assert group.world_size == world_size
            _check(lib().fpdt_ctx_create_local(group.handle, rank, device, host_arena_bytes, ctypes.byref(h)))
        else:
            _check(lib().fpdt_ctx_create(world_size, rank, nccl_id, device, host_arena_bytes, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            _check(lib().fpdt_ctx_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = Stats()
        _check(lib().fpdt_get_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()

    def set_sparsity(self, keep=None):
        """Block-sparsity plan keep [u, u] (numpy bool/uint8; None = dense) for the following forward calls."""
        if keep is None:
            _check(lib().fpdt_set_sparsity(self.handle, None, 0))
            return
        import numpy as np
        k = np.ascontiguousarray(np.asarray(keep, dtype=np.uint8))
        assert k.ndim == 2 and k.shape[0] == k.shape[1]
        self._plan = k  # keep alive during the call (the library copies it)
        _check(lib().fpdt_set_sparsity(self.handle, c_void_p(k.ctypes.data), k.shape[0]))

    def set_residency(self, kv_chunks: int = 0, q_chunks: int = 0):
        """HBM residency budget for the following forward calls (offload = 1): key/value chunks i < kv_chunks and
        query-side chunks i >= u - q_chunks stay in device memory (include/fpdt.h)."""
        _check(lib().fpdt_set_residency(self.handle, int(kv_chunks), int(q_chunks)))

    def set_hidden_offload(self, enable: bool = True):
        """fpdt_block_fwd offloads the hidden-state chunks; fpdt_block_bwd may then take x = None."""
        _check(lib().fpdt_set_hidden_offload(self.handle, int(enable)))

    def set_fetch_strategy(self, strategy: int):
        """FPDT_FETCH_PER_RANK (A) or FPDT_FETCH_LEADER (B, rank 0 fetches and scatters)."""
        _check(lib().fpdt_set_fetch_strategy(self.handle, int(strategy)))

    def set_debug_checks(self, enable: bool = True):
        _check(lib().fpdt_set_debug_checks(self.handle, int(enable)))

    def set_bwd_order(self, order: int):
        """Backward loop order for the following backward calls: FPDT_BWD_KV_OUTER (the paper's), FPDT_BWD_Q_OUTER
        (GQA-aware: the dK/dV partials round-trip the host instead of the dq partials) or FPDT_BWD_AUTO
        (include/fpdt.h)."""
        _check(lib().fpdt_set_bwd_order(self.handle, int(order)))

    def set_kernel_timing(self, enable: bool):
        _check(lib().fpdt_set_kernel_timing(self.handle, int(enable)))

    def kernel_time(self, reset: bool = True):
        f, b = ctypes.c_double(), ctypes.c_double()
        nf, nb = c_int64(), c_int64()
        _check(lib().fpdt_kernel_time(self.handle, ctypes.byref(f), ctypes.byref(nf), ctypes.byref(b),
                                      ctypes.byref(nb), int(reset)))
        return f.value, nf.value, b.value, nb.value

    def exchange_time(self):
        """dict(total_ms, n, bytes, first_ms, last_ms) of the all-to-alls since the last kernel_time reset."""
        t, f, l = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        n, b = c_int64(), c_int64()
        _check(lib().fpdt_exchange_time(self.handle, ctypes.byref(t), ctypes.byref(n), ctypes.byref(b), ctypes.byref(f),
                                        ctypes.byref(l)))
        return {"total_ms": t.value, "n": n.value, "bytes": b.value, "first_ms": f.value, "last_ms": l.value}

    def kernel_gaps(self):
        """(gap_ms, n_gaps): compute-stream time between consecutive attention launches of one call since the last
        kernel_time reset (include/fpdt.h fpdt_kernel_gaps)."""
        g, n = ctypes.c_double(), c_int64()
        _check(lib().fpdt_kernel_gaps(self.handle, ctypes.byref(g), ctypes.byref(n)))
        return g.value, n.value


def fpdt_attn_fwd(ctx: FPDTContext, q, k, v, o, lse, s_local: int, n_q_heads: int, n_kv_heads: int, head_dim: int,
                  causal: int, chunk_size: int, world_size: int, dtype: int, offload: int,
                  softmax_scale: float = 0.0, stream=None):
    _check(lib().fpdt_attn_fwd(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), s_local, n_q_heads,
                               n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload, softmax_scale,
                               _stream(stream)))


def fpdt_attn_bwd(ctx: FPDTContext, o, dout, dq, dk, dv, s_local: int, n_q_heads: int, n_kv_heads: int,
                  head_dim: int, causal: int, chunk_size: int, world_size: int, dtype: int, offload: int,
                  softmax_scale: float = 0.0, stream=None):
    _check(lib().fpdt_attn_bwd(ctx.handle, _ptr(o), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv), s_local, n_q_heads,
                               n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload, softmax_scale,
                               _stream(stream)))


def fpdt_attn_fwd_host(ctx: FPDTContext, q, k, v, o, lse, s_local: int, n_q_heads: int, n_kv_heads: int,
                       head_dim: int, causal: int, chunk_size: int, world_size: int, dtype: int, offload: int,
                       softmax_scale: float = 0.0, stream=None):
    """q, k, v, o, lse: pinned host tensors (include/fpdt.h fpdt_attn_fwd_host)."""
    _check(lib().fpdt_attn_fwd_host(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), s_local, n_q_heads,
                                    n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                                    softmax_scale, _stream(stream)))


def fpdt_attn_bwd_host(ctx: FPDTContext, o, dout, dq, dk, dv, s_local: int, n_q_heads: int, n_kv_heads: int,
                       head_dim: int, causal: int, chunk_size: int, world_size: int, dtype: int, offload: int,
                       softmax_scale: float = 0.0, stream=None):
    """o, dout, dq, dk, dv: pinned host tensors (include/fpdt.h fpdt_attn_bwd_host)."""
    _check(lib().fpdt_attn_bwd_host(ctx.handle, _ptr(o), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv), s_local,
                                    n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload,
                                    softmax_scale, _stream(stream)))


def fpdt_block_fwd(ctx: FPDTContext, x, w_qkv, o, lse, s_local: int, hidden: int, n_q_heads: int, n_kv_heads: int,
                   head_dim: int, causal: int, chunk_size: int, world_size: int, dtype: int, offload: int,
                   softmax_scale: float = 0.0, stream=None, w_o=None, y=None):
    _check(lib().fpdt_block_fwd(ctx.handle, _ptr(x), _ptr(w_qkv), _ptr(w_o), _ptr(o), _ptr(lse), _ptr(y), s_local,
                                hidden, n_q_heads,
                                n_kv_heads, head_dim, causal, chunk_size, world_size, dtype, offload, softmax_scale,
                                _stream(stream)))


def fpdt_block_bwd(ctx: FPDTContext, x, w_qkv, o, dout, dx, dw_qkv, s_local: int, hidden: int, n_q_heads: int,
                   n_kv_heads: int, head_dim: int, causal: int, chunk_size: int, world_size: int, dtype: int,
                   offload: int, softmax_scale: float = 0.0, stream=None, w_o=None, dw_o=None):
    """dout: dL/do, or dL/dy [s_local, hidden] when w_o is given (include/fpdt.h)."""
    _check(lib().fpdt_block_bwd(ctx.handle, _ptr(x), _ptr(w_qkv), _ptr(w_o), _ptr(o), _ptr(dout), _ptr(dx),
                                _ptr(dw_qkv), _ptr(dw_o),
                                s_local, hidden, n_q_heads, n_kv_heads, head_dim, causal, chunk_size, world_size,
                                dtype, offload, softmax_scale, _stream(stream)))


def fpdt_bwd_host_bytes(order: int, s_local: int, n_q_heads: int, n_kv_heads: int, head_dim: int, chunk_size: int,
                        world_size: int, dtype: int, kv_chunks: int = 0, q_chunks: int = 0, keep=None) -> int:
    """Host-link bytes of the backward chunk loop in `order` (the model FPDT_BWD_AUTO compares; host-only)."""
    out = c_int64()
    plan, n = None, 0
    if keep is not None:
        import numpy as np
        plan = np.ascontiguousarray(np.asarray(keep, dtype=np.uint8))
        n = plan.shape[0]
    _check(lib().fpdt_bwd_host_bytes(order, s_local, n_q_heads, n_kv_heads, head_dim, chunk_size, world_size, dtype,
                                     kv_chunks, q_chunks, None if plan is None else c_void_p(plan.ctypes.data), n,
                                     ctypes.byref(out)))
    return out.value


def dtype_code(torch_dtype) -> int:
    import torch
    if torch_dtype == torch.bfloat16:
        return FPDT_BF16
    if torch_dtype == torch.float32:
        return FPDT_FP32
    raise FpdtError(FPDT_ERR_UNSUPPORTED, f"dtype {torch_dtype}")
