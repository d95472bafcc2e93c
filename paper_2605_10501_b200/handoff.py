"""K5b handoff (scatter) indices on device and the K6 row moves that use them.

A producer section (modality encoder, or the teacher) writes ``rows[i]`` output rows per sample
``i`` into one row buffer, in its own (fan-out merged) schedule order; the consumer (critical)
rank packs its samples in its order into micro-batches (``maestro_varlen_pack``).
:func:`handoff_index` computes on device, from those orders alone, every (producer row,
consumer row) pair -- the placeholder positions of PAPER.md:56,250 -- so no per-micro-batch
index is built on the host (include/maestro_b200.h: maestro_handoff_index).  The CPU restatement
the tests compare with bit-exactly is ``oracle/handoff_ref.py``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N

_P, _I32 = ctypes.c_void_p, ctypes.c_int32
_L = None


def _lib():
    global _L
    if _L is None:
        _L = N.extra_symbols({
            "maestro_handoff_index": ([_P, _I32, _P, _I32, _P, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P],
                                      ctypes.c_int),
            "maestro_scatter_rows_range": ([_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P], ctypes.c_int),
        })
    return _L


@dataclass
class HandoffIndex:
    """Device index of one producer -> consumer edge for one step: ``pos`` [n+1] (exclusive scan
    of rows over the consumer order), ``src`` / ``dst`` [total] row pairs; ``mbs`` the consumer
    micro-batch size, ``n`` its samples."""

    pos: torch.Tensor
    src: torch.Tensor
    dst: torch.Tensor
    mbs: int
    n: int
    max_rows_mb: int   # host bound on the rows of one consumer micro-batch (grid sizing)

    def mb_range(self, m: int) -> tuple[int, int]:
        return m * self.mbs, min(self.n, (m + 1) * self.mbs)


def handoff_index(up_order: torch.Tensor, crit_order: torch.Tensor, tok_off: torch.Tensor, mbs: int,
                  rows: torch.Tensor, dst_off: torch.Tensor, total_rows: int, max_rows_mb: int,
                  err: torch.Tensor | None = None) -> HandoffIndex:
    """All int32 device tensors; ``rows`` / ``dst_off`` are indexed by sample id (length B).
    ``total_rows`` >= sum of rows over the consumer order (allocation bound)."""
    dev = crit_order.device
    B, n, nu = rows.numel(), crit_order.numel(), up_order.numel()
    scratch = torch.empty(B, dtype=torch.int32, device=dev)
    pos = torch.empty(n + 1, dtype=torch.int32, device=dev)
    src = torch.empty(max(total_rows, 1), dtype=torch.int32, device=dev)
    dst = torch.empty(max(total_rows, 1), dtype=torch.int32, device=dev)
    N.check(_lib().maestro_handoff_index(N.ptr(up_order), nu, N.ptr(crit_order), n, N.ptr(tok_off), mbs,
                                         N.ptr(rows), N.ptr(dst_off), B, N.ptr(scratch), N.ptr(pos), N.ptr(src),
                                         N.ptr(dst), N.ptr(err) if err is not None else None, N.stream_ptr()),
            "handoff_index")
    return HandoffIndex(pos, src, dst, mbs, n, max_rows_mb)


def scatter_mb(ix: HandoffIndex, m: int, src_buf: torch.Tensor, dst_buf: torch.Tensor, reverse: bool = False,
               accumulate: bool = False):
    """K6 for consumer micro-batch m: dst_buf[dst] = src_buf[src] (reverse: the other direction,
    dst_buf[src] = src_buf[dst]; accumulate: += instead of =).  The pair range stays on device."""
    k0, k1 = ix.mb_range(m)
    a, b = (ix.dst, ix.src) if reverse else (ix.src, ix.dst)
    N.check(_lib().maestro_scatter_rows_range(N.ptr(src_buf), N.ptr(dst_buf), N.ptr(a), N.ptr(b), N.ptr(ix.pos), k0,
                                              k1, ix.max_rows_mb, src_buf.shape[-1], int(accumulate),
                                              N.stream_ptr()), "scatter_rows_range")
