"""C2 overlapped with the backward: a section's gradient all-reduce in per-layer buckets.

Gradients accumulate over a section's micro-batches, so a layer's gradient is final once the LAST
micro-batch's backward has passed it.  During that backward, ``layer_done(i)`` (the
``Transformer.backward`` layer hook) records an event on the compute stream and enqueues the
all-reduce of layer i's slice of the flat gradient arena on a communication stream, so the
reductions of layers L-1 .. 0 run while the backward continues towards layer 0; ``finish``
reduces the remaining slices (embedding, final norm, head, projector weights -- their gradients
complete at the end) and joins the streams before the optimizer.  While buckets are in flight,
persistent compute grids leave ``reserve`` SMs to NCCL's kernels (maestro_set_sm_budget), so a
persistent tile schedule never waits on a CTA that NCCL keeps from becoming resident.
"""

from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _native as N
from .transformer import _align


def _subtract(ranges, holes):
    """[a, b) ranges minus the hole ranges (each hole inside one range)."""
    out = list(ranges)
    for h0, h1 in holes:
        nxt = []
        for a, b in out:
            if h1 <= a or h0 >= b:
                nxt.append((a, b))
                continue
            if a < h0:
                nxt.append((a, h0))
            if h1 < b:
                nxt.append((h1, b))
        out = nxt
    return out


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


class GradSync:
    def __init__(self, params, n_layers: int, group=None, device=None, reserve: int = 8):
        self.p = params
        idx = params.index
        self.layers = []
        for i in range(n_layers):
            a = idx[f"l{i}.ln1"][0]
            o, shp = idx[f"l{i}.wd"]
            self.layers.append((a, o + _align(math.prod(shp))))
        lo, hi = (self.layers[0][0], self.layers[-1][1]) if self.layers else (0, 0)
        rest = [(a, b) for a, b in ((0, lo), (hi, params.numel)) if b > a]
        # the untied output head and the final norm are final right after their (first) backward
        # step: reduced at layer_done(-1), not with the embedding at the end (MAESTRO_C2_EARLY_HEAD)
        self.early = []
        if "head" in idx and os.environ.get("MAESTRO_C2_EARLY_HEAD", "1") != "0":
            for name in ("head", "lnf"):
                o, shp = idx[name]
                self.early.append((o, o + _align(math.prod(shp))))
        self.rest = _subtract(rest, self.early)
        self.group = group
        self.comm = torch.cuda.Stream(device=device)
        self.reserve = reserve
        self.pending = set()
        self._budget_set = False
        self._sms = torch.cuda.get_device_properties(device or torch.cuda.current_device()).multi_processor_count

    def _budget(self, n: int) -> None:
        L = N.extra_symbols({"maestro_set_sm_budget": ([ctypes.c_int32], ctypes.c_int)})
        N.check(L.maestro_set_sm_budget(n), "set_sm_budget")

    def begin(self) -> None:
        """Before the last micro-batch's backward: every layer is pending; compute grids shrink."""
        self.pending = set(range(len(self.layers))) | ({-1} if self.early else set())
        if self.reserve > 0:
            self._budget(self._sms - self.reserve)
            self._budget_set = True

    def _reduce(self, a: int, b: int) -> None:
        _dist().all_reduce(self.p.grad[a:b], group=self.group)

    def layer_done(self, i: int) -> None:
        """Layer hook: layer i's gradient is final on the current stream -> reduce it on comm
        (i = -1: the output head and final norm, before the layers)."""
        if i not in self.pending:
            return
        self.pending.discard(i)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            for a, b in (self.early if i == -1 else [self.layers[i]]):
                self._reduce(a, b)

    def finish(self, stream) -> None:
        """After the backward: reduce what is left and make ``stream`` wait for every bucket."""
        if self._budget_set:
            self._budget(0)
            self._budget_set = False
        ev = torch.cuda.Event()
        ev.record(stream)
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            for i in sorted(self.pending):
                for a, b in (self.early if i == -1 else [self.layers[i]]):
                    self._reduce(a, b)
            for a, b in self.rest:
                self._reduce(a, b)
        self.pending = set()
        stream.wait_stream(self.comm)
