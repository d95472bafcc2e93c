"""Thin typed wrappers over the memory-bound kernels of the C ABI (csrc/elementwise.cu, kd_loss.cu).

Every function takes torch CUDA tensors, launches on the current stream and returns
immediately.  The native library is mandatory (see _native.lib()).
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from . import instrument

_P, _I32, _I64, _F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
_SIGS = {
    "maestro_add_rmsnorm_fwd": [_P, _P, _P, _P, _P, _P, _I32, _I32, _F, _P],
    "maestro_rmsnorm_bwd": [_P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P],
    "maestro_rope": [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P],
    "maestro_positions": [_P, _I32, _P, _P],
    "maestro_swiglu_fwd": [_P, _P, _I32, _I32, _P],
    "maestro_swiglu_bwd": [_P, _P, _P, _I32, _I32, _P],
    "maestro_embed_fwd": [_P, _P, _P, _I32, _I32, _P],
    "maestro_embed_bwd": [_P, _P, _P, _I32, _I32, _P],
    "maestro_transpose_bf16": [_P, _P, _I32, _I32, _I32, _I32, _P],
    "maestro_transpose_bf16_batched": [_P, _I32, _I32, _P],
    "maestro_adamw": [_P, _P, _P, _P, _P, _I64, _F, _F, _F, _F, _F, _I32, _F, _P],
    "maestro_kd_loss_fwd_bwd": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _F, _F, _P],
    "maestro_ce_loss_fwd_bwd": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _F, _P],
    "maestro_scatter_rows_fwd": [_P, _P, _P, _P, _I32, _I32, _P],
    "maestro_gather_rows_bwd": [_P, _P, _P, _P, _I32, _I32, _P],
}
_L = None


def L():
    global _L
    if _L is None:
        _L = N.extra_symbols({k: (v, ctypes.c_int) for k, v in _SIGS.items()})
    return _L


def _p(t):
    return None if t is None else t.data_ptr()


def _s():
    return N.stream_ptr()


def add_rmsnorm(x, a, h, y, w, rstd, eps=1e-5):
    """h = x + a (skipped when a is None); y = rmsnorm(h) * w; rstd[T] saved for backward."""
    T, d = x.shape
    N.check(L().maestro_add_rmsnorm_fwd(_p(x), _p(a), _p(h), _p(y), _p(w), _p(rstd), T, d, eps, _s()), "rmsnorm_fwd")


def rmsnorm_bwd(dy, h, w, rstd, dres, dx, dw):
    """dx = dres + d rmsnorm(h)/dh . dy;  dw (fp32) += sum_rows dy * h * rstd."""
    T, d = dy.shape
    N.check(L().maestro_rmsnorm_bwd(_p(dy), _p(h), _p(w), _p(rstd), _p(dres), _p(dx), _p(dw), T, d, _s()),
            "rmsnorm_bwd")


def rope(qk, pos, cos_sin, n_heads, dh, backward=False):
    """In-place rotate-half RoPE on ``qk`` rows ([T, n_heads*dh] view with row pitch)."""
    T = qk.shape[0]
    N.check(L().maestro_rope(_p(qk), _p(pos), _p(cos_sin), T, n_heads, dh, qk.stride(0), int(backward), _s()),
            "rope")


def positions(cu, nseq, pos):
    N.check(L().maestro_positions(_p(cu), nseq, _p(pos), _s()), "positions")


def swiglu(gu, out):
    T, F2 = gu.shape
    N.check(L().maestro_swiglu_fwd(_p(gu), _p(out), T, F2 // 2, _s()), "swiglu_fwd")


def swiglu_bwd(dout, gu, dgu):
    T, F2 = gu.shape
    N.check(L().maestro_swiglu_bwd(_p(dout), _p(gu), _p(dgu), T, F2 // 2, _s()), "swiglu_bwd")


def embed(table, ids, out):
    T, d = out.shape
    N.check(L().maestro_embed_fwd(_p(table), _p(ids), _p(out), T, d, _s()), "embed_fwd")


def embed_bwd(dout, ids, dtable):
    T, d = dout.shape
    N.check(L().maestro_embed_bwd(_p(dout), _p(ids), _p(dtable), T, d, _s()), "embed_bwd")


def transpose(src, dst):
    """dst[c, r] = src[r, c] (bf16, 2-D, row pitch from the tensors)."""
    R, C = src.shape
    N.check(L().maestro_transpose_bf16(_p(src), _p(dst), R, C, src.stride(0), dst.stride(0), _s()), "transpose_bf16")


def transpose_batch_desc(pairs, device) -> tuple[torch.Tensor, int]:
    """Descriptor table for transpose_batched: pairs = [(src, dst)] of 2-D bf16 tensors (dst is
    src^T).  Returns (int64 [n, 8] on device, total tiles).  Pointers are captured: rebuild if
    any tensor is reallocated."""
    rows, first = [], 0
    for src, dst in pairs:
        R, C = src.shape
        if R % 8 or C % 8 or src.stride(0) % 8 or dst.stride(0) % 8:
            raise ValueError("transpose_batched: rows, cols and pitches must be multiples of 8")
        tx, ty = (C + 63) // 64, (R + 63) // 64
        rows.append([src.data_ptr(), dst.data_ptr(), R, C, src.stride(0), dst.stride(0), first, tx])
        first += tx * ty
    return torch.tensor(rows, dtype=torch.int64, device=device), first


def transpose_batched(desc: torch.Tensor, total_tiles: int):
    """All transposes of a transpose_batch_desc table in one launch."""
    N.check(L().maestro_transpose_bf16_batched(_p(desc), desc.shape[0], total_tiles, _s()), "transpose_batched")


def adamw(p, g, m, v, pb, lr, step, b1=0.9, b2=0.95, eps=1e-8, wd=0.1, gscale=1.0):
    N.check(L().maestro_adamw(_p(p), _p(g), _p(m), _p(v), _p(pb), p.numel(), lr, b1, b2, eps, wd, step, gscale,
                              _s()), "adamw")


def kd_loss(t_logits, s_logits, ds, loss, grad_scale, tau=1.0):
    """Fused full-vocab KL(teacher || student) per token + d/ds (K9).  ds may be s_logits."""
    T, V = s_logits.shape
    tok = instrument.begin("kd_loss", 2.0 * T * V * (3 if ds is not None else 2))  # read t, s (+ write ds)
    N.check(L().maestro_kd_loss_fwd_bwd(_p(t_logits), _p(s_logits), _p(ds), _p(loss), T, V, t_logits.stride(0),
                                        s_logits.stride(0), ds.stride(0) if ds is not None else 8, grad_scale,
                                        1.0 / tau, _s()), "kd_loss")
    instrument.end(tok)


def ce_loss(logits, labels, ds, loss, grad_scale):
    """Fused full-vocab next-token cross entropy (+ d/dlogits); labels < 0 are ignored."""
    T, V = logits.shape
    N.check(L().maestro_ce_loss_fwd_bwd(_p(logits), _p(labels), _p(ds), _p(loss), T, V, logits.stride(0),
                                        ds.stride(0), grad_scale, _s()), "ce_loss")


def scatter_rows(src, dst, src_rows, dst_rows):
    """K6: dst[dst_rows[k]] = src[src_rows[k]] (bf16 rows, 16-byte vectors)."""
    n = src_rows.numel()
    N.check(L().maestro_scatter_rows_fwd(_p(src), _p(dst), _p(src_rows), _p(dst_rows), n, src.shape[-1], _s()),
            "scatter_rows")


def gather_rows_bwd(ddst, dsrc, seg, seg_dst):
    """K6 backward: dsrc[r] = sum_{k in seg[r]..seg[r+1]} ddst[seg_dst[k]] (fp32 accumulate)."""
    N.check(L().maestro_gather_rows_bwd(_p(ddst), _p(dsrc), _p(seg), _p(seg_dst), dsrc.shape[0], dsrc.shape[-1],
                                        _s()), "gather_rows_bwd")
