"""Varlen (packed, cu_seqlens) attention with GQA on tcgen05/TMEM (K8, csrc/attention.cu).

Layout: q [T, H, dh], k/v [T, Hkv, dh] (row-pitched views into the fused QKV buffer),
o [T, H, dh] bf16, lse [H, T] fp32 (natural log-sum-exp of the scaled scores).  The backward
writes dq/dk/dv straight into the fused dQKV buffer views.  head_dim 64 or 128.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from . import instrument

_P, _I32, _F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float
_bound = None


def _lib():
    global _bound
    if _bound is None:
        _bound = N.extra_symbols({
            "maestro_attn_workspace": ([_I32, _I32], ctypes.c_int64),
            "maestro_attn_bwd_workspace": ([_I32, _I32, _I32, _I32], ctypes.c_int64),
            "maestro_attn_plan_size": ([_I32, _I32], ctypes.c_int64),
            "maestro_attn_plan": ([_P, _I32, _I32, _P, _P], ctypes.c_int),
            "maestro_attn_fwd": ([_P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _F,
                                  _I32, _P, _P, _P], ctypes.c_int),
            "maestro_attn_bwd": ([_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                                  _I32, _P, _I32, _P, _I32, _P, _I32, _F, _I32, _P, _P, _P, _P, _P], ctypes.c_int),
        })
    return _bound


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty((nbytes + 255) // 256 * 256, dtype=torch.uint8, device=device)


def plan(cu, T: int) -> torch.Tensor:
    """Work plan of one packed micro-batch (tile lists), shared by every layer's fwd/bwd."""
    L = _lib()
    nseq = cu.numel() - 1
    buf = _ws(L.maestro_attn_plan_size(T, nseq), cu.device)
    N.check(L.maestro_attn_plan(cu.data_ptr(), nseq, T, buf.data_ptr(), N.stream_ptr()), "attn_plan")
    return buf


def attn_fwd(q, k, v, cu, max_len: int, causal: bool, out, scale: float, plan=None):
    """Writes out [T, H, dh]; returns lse [H, T] fp32.  ``plan``: attention.plan(cu, T) or None."""
    L = _lib()
    T, H, dh = q.shape
    Hk = k.shape[1]
    nseq = cu.numel() - 1
    lse = torch.empty(H, T, dtype=torch.float32, device=q.device)
    ws = _ws(L.maestro_attn_workspace(T, nseq), q.device)
    tok = instrument.begin("attn_fwd")
    rc = L.maestro_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), cu.data_ptr(), nseq, T, H, Hk, dh,
                            q.stride(0), k.stride(0), v.stride(0), out.data_ptr(), out.stride(0), lse.data_ptr(),
                            scale, int(causal), plan.data_ptr() if plan is not None else None, ws.data_ptr(),
                            N.stream_ptr())
    N.check(rc, "attn_fwd")
    instrument.end(tok)
    return lse


def attn_bwd(do, q, k, v, o, lse, cu, max_len: int, causal: bool, dq, dk, dv, scale: float, rope=None, plan=None):
    """rope=(pos, cos_sin): dq/dk come back through the inverse RoPE rotation (fused)."""
    L = _lib()
    T, H, dh = q.shape
    Hk = k.shape[1]
    nseq = cu.numel() - 1
    ws = _ws(L.maestro_attn_bwd_workspace(T, nseq, H, dh), q.device)
    tok = instrument.begin("attn_bwd")
    rc = L.maestro_attn_bwd(do.data_ptr(), do.stride(0), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                            o.stride(0), lse.data_ptr(), cu.data_ptr(), nseq, T, H, Hk, dh, q.stride(0), k.stride(0),
                            v.stride(0), dq.data_ptr(), dq.stride(0), dk.data_ptr(), dk.stride(0), dv.data_ptr(),
                            dv.stride(0), scale, int(causal), rope[0].data_ptr() if rope else None,
                            rope[1].data_ptr() if rope else None, plan.data_ptr() if plan is not None else None,
                            ws.data_ptr(), N.stream_ptr())
    N.check(rc, "attn_bwd")
    instrument.end(tok)
