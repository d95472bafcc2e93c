"""Host wrappers of the tcgen05 GEMM (K7, csrc/gemm.cu) for the three training GEMMs.

All tensors are torch CUDA tensors (bf16 operands; fp32 or bf16 outputs).  No
autograd and no cuBLAS: the section compute calls these directly with explicit
forward / dgrad / wgrad.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from . import instrument

EPI_BF16, EPI_F32, EPI_F32_ACC = 0, 1, 2

_bound = False


def _lib():
    global _bound
    L = N.lib()
    if not _bound:
        I32, P = ctypes.c_int32, ctypes.c_void_p
        N.extra_symbols({
            "maestro_gemm_bf16": ([P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, P], ctypes.c_int),
            "maestro_gemm_bf16_rope": ([P, P, P, I32, I32, I32, I32, I32, I32, P, P, I32, I32, P], ctypes.c_int),
            "maestro_gemm_bf16_swiglu": ([P, P, P, I32, I32, I32, I32, I32, I32, P, I32, P], ctypes.c_int),
            "maestro_gemm_bf16_residual": ([P, P, P, I32, I32, I32, I32, I32, I32, P, I32, P], ctypes.c_int),
        })
        _bound = True
    return L


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, M: int, N_: int, K: int, a_mn: bool, b_mn: bool,
         epi: int, lda: int | None = None, ldb: int | None = None, ldc: int | None = None) -> torch.Tensor:
    """c[m, n] (+)= sum_k A(m,k) B(n,k); see include/maestro_b200.h (maestro_gemm_bf16)."""
    if lda is None:
        lda = a.stride(0)
    if ldb is None:
        ldb = b.stride(0)
    if ldc is None:
        ldc = c.stride(0)
    rec = instrument.gemm_timing
    if rec is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = _lib().maestro_gemm_bf16(N.ptr(a), N.ptr(b), N.ptr(c), M, N_, K, lda, ldb, ldc, int(a_mn), int(b_mn),
                                  epi, N.stream_ptr())
    N.check(rc, "gemm_bf16")
    if rec is not None:
        e1.record()
        rec.append((2.0 * M * N_ * K, e0, e1))
    return c


def linear_fwd(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """y[T, out] = x[T, in] @ w[out, in]^T."""
    T, K = x.shape
    Nn = w.shape[0]
    if out is None:
        out = torch.empty(T, Nn, device=x.device, dtype=torch.bfloat16)
    return gemm(x, w, out, T, Nn, K, False, False, EPI_BF16)


def linear_fwd_rope(x: torch.Tensor, w: torch.Tensor, pos: torch.Tensor, cos_sin: torch.Tensor, rope_cols: int,
                    out: torch.Tensor | None = None, head_dim: int = 64) -> torch.Tensor:
    """qkv = x @ w^T with RoPE applied to the ``head_dim``-wide heads (64 or 128) of the first
    ``rope_cols`` columns inside the GEMM epilogue."""
    T, K = x.shape
    Nn = w.shape[0]
    if out is None:
        out = torch.empty(T, Nn, device=x.device, dtype=torch.bfloat16)
    rec = instrument.gemm_timing
    if rec is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = _lib().maestro_gemm_bf16_rope(N.ptr(x), N.ptr(w), N.ptr(out), T, Nn, K, x.stride(0), w.stride(0),
                                       out.stride(0), N.ptr(pos), N.ptr(cos_sin), rope_cols, head_dim,
                                       N.stream_ptr())
    N.check(rc, "gemm_bf16_rope")
    if rec is not None:
        e1.record()
        rec.append((2.0 * T * Nn * K, e0, e1))
    return out


def linear_fwd_residual(x: torch.Tensor, w: torch.Tensor, resid: torch.Tensor,
                        out: torch.Tensor | None = None) -> torch.Tensor:
    """h[T, out] = resid + x @ w^T (residual add fused into the GEMM epilogue)."""
    T, K = x.shape
    Nn = w.shape[0]
    if out is None:
        out = torch.empty(T, Nn, device=x.device, dtype=torch.bfloat16)
    rec = instrument.gemm_timing
    if rec is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = _lib().maestro_gemm_bf16_residual(N.ptr(x), N.ptr(w), N.ptr(out), T, Nn, K, x.stride(0), w.stride(0),
                                           out.stride(0), N.ptr(resid), resid.stride(0), N.stream_ptr())
    N.check(rc, "gemm_bf16_residual")
    if rec is not None:
        e1.record()
        rec.append((2.0 * T * Nn * K, e0, e1))
    return out


def linear_fwd_swiglu(x: torch.Tensor, w: torch.Tensor, s_out: torch.Tensor,
                      out: torch.Tensor | None = None, store_gu: bool = True) -> torch.Tensor | None:
    """gu = x @ w^T (gate/up interleaved in 32-row blocks) and s_out = silu(g) * u from the epilogue.
    ``store_gu=False`` (forward-only sections) writes only s_out and returns None."""
    T, K = x.shape
    Nn = w.shape[0]
    if out is None and store_gu:
        out = torch.empty(T, Nn, device=x.device, dtype=torch.bfloat16)
    rec = instrument.gemm_timing
    if rec is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = _lib().maestro_gemm_bf16_swiglu(N.ptr(x), N.ptr(w), N.ptr(out) if out is not None else None, T, Nn, K,
                                         x.stride(0), w.stride(0), out.stride(0) if out is not None else Nn,
                                         N.ptr(s_out), s_out.stride(0), N.stream_ptr())
    N.check(rc, "gemm_bf16_swiglu")
    if rec is not None:
        e1.record()
        rec.append((2.0 * T * Nn * K, e0, e1))
    return out


def linear_dgrad(dy: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None,
                 wt: torch.Tensor | None = None) -> torch.Tensor:
    """dx[T, in] = dy[T, out] @ w[out, in].  ``wt`` = w^T [in, out] (bf16) makes B K-major."""
    T, Nn = dy.shape
    K = w.shape[1]
    if out is None:
        out = torch.empty(T, K, device=dy.device, dtype=torch.bfloat16)
    if wt is not None:
        return gemm(dy, wt, out, T, K, Nn, False, False, EPI_BF16, ldb=wt.stride(0))
    return gemm(dy, w, out, T, K, Nn, False, True, EPI_BF16, ldb=w.stride(0))


def linear_wgrad(dy: torch.Tensor, x: torch.Tensor, dw: torch.Tensor, accumulate: bool = True) -> torch.Tensor:
    """dw[out, in] (+)= dy[T, out]^T @ x[T, in]   (dw fp32)."""
    T, Nn = dy.shape
    K = x.shape[1]
    return gemm(dy, x, dw, Nn, K, T, True, True, EPI_F32_ACC if accumulate else EPI_F32,
                lda=dy.stride(0), ldb=x.stride(0))
