"""Varlen (packed, cu_seqlens) causal / bidirectional attention with GQA: forward + backward.

Layout: q [T, H, dh], k/v [T, Hkv, dh] (row-pitched views into the fused QKV buffer),
o [T, H, dh] bf16, lse [H, T] fp32 (natural log of the softmax denominator of the scaled
scores).  Backward writes dq/dk/dv into the fused dQKV buffer views.

Round-1 status: the forward/backward are served by the flash-attn 2 library kernels
(sm_100 build shipped in the image), wrapped behind this interface; the hand-written
tcgen05/TMEM replacement (csrc/attention.cu) is the next kernel in DESIGN.md and plugs in
here without touching the callers.
"""

from __future__ import annotations

import torch

_fa = None


def _lib():
    global _fa
    if _fa is None:
        from flash_attn import flash_attn_interface as fa

        _fa = fa
    return _fa


def attn_fwd(q, k, v, cu, max_len: int, causal: bool, out, scale: float):
    """Returns lse [H, T] fp32; writes out."""
    fa = _lib()
    o, lse, _, _ = fa._flash_attn_varlen_forward(q, k, v, cu, cu, max_len, max_len, 0.0, scale, causal)
    out.copy_(o)
    return lse


def attn_bwd(do, q, k, v, o, lse, cu, max_len: int, causal: bool, dq, dk, dv, scale: float):
    fa = _lib()
    dq_, dk_, dv_ = (torch.empty(t.shape, device=t.device, dtype=t.dtype) for t in (dq, dk, dv))
    fa._flash_attn_varlen_backward(do.contiguous(), q, k, v, o, lse, dq_, dk_, dv_, cu, cu, max_len, max_len, 0.0,
                                   scale, causal, -1, -1, 0.0, None, False)
    dq.copy_(dq_)
    dk.copy_(dk_)
    dv.copy_(dv_)
