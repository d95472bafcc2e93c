"""Wavefront scheduler API, backed by the device kernels K1-K4 (csrc/plan.cu).

Same entry points, argument meaning and exceptions as the reference
(``maestro/scheduling.py``): ``ExecPolicy`` (:39-53), ``RankMetrics`` (:56-66),
``EvalCounter`` (:69-73), ``sort_initial`` (:76-78), ``rank_metrics``
(:81-152), ``calculate_makespan`` (:155-159), ``schedule_rank`` (:162-199),
``partition_batch`` (:202-264), ``merge_fanout`` (:267-285), ``Schedule``
(:288-306) and ``build_schedule`` (:309-373).  The arithmetic runs on the GPU
and is bit-identical to the reference's fp64 results.

:class:`DevicePlanner` is the allocation-free, stream-ordered form used by the
executor every step: it keeps the batch, the plan and the error word in HBM
and never synchronises; the Python functions above it are the synchronous
convenience layer that returns Python objects.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Mapping, Optional, Sequence, TypeVar

import numpy as np

from . import _native as N
from .errors import EmptyBatch, FanoutMismatch, InconsistentSchedule, NativeError
from .workload import PHASES, SampleTiming, SectionConfig, SectionGraph, SectionId

T = TypeVar("T")


class ExecPolicy(str, Enum):
    """Forward/backward interleave of the critical and downstream resources."""

    INTERLEAVED = "interleaved"
    ALL_FWD_THEN_BWD = "all-fwd-then-bwd"

    @classmethod
    def parse(cls, value) -> "ExecPolicy":
        if isinstance(value, ExecPolicy):
            return value
        try:
            return cls(value)
        except ValueError:
            raise ValueError(f"unknown exec policy '{value}' (options: {', '.join(p.value for p in cls)})")

    @property
    def code(self) -> int:
        return 0 if self is ExecPolicy.INTERLEAVED else 1


@dataclass(frozen=True)
class RankMetrics:
    makespan: float
    critical_busy: float
    critical_span: float

    @property
    def critical_idle(self) -> float:
        """Section stall of the critical rank: span - busy (scheduling.py:64-66)."""
        return self.critical_span - self.critical_busy


@dataclass
class EvalCounter:
    count: int = 0


@dataclass(frozen=True)
class Schedule:
    """Per-(section, dp_rank) sample-id orders plus the batch (scheduling.py:288-306)."""

    per_rank_orders: Mapping[tuple[SectionId, int], tuple[int, ...]]
    batch: tuple[SampleTiming, ...]
    policy: ExecPolicy = ExecPolicy.INTERLEAVED

    def order_for(self, section: SectionId, rank: int) -> tuple[int, ...]:
        return self.per_rank_orders.get((section, rank), ())

    def ranks_of(self, section: SectionId) -> list[int]:
        return sorted(r for (sec, r) in self.per_rank_orders if sec == section)

    def sample(self, sample_id: int) -> SampleTiming:
        for s in self.batch:
            if s.sample_id == sample_id:
                return s
        raise InconsistentSchedule(f"schedule references unknown sample {sample_id}")


# ----------------------------------------------------------------------------- device helpers
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("a CUDA device (B200, sm_100a) is required; there is no CPU path")
    return torch


def _times_host(samples: Sequence[SampleTiming]) -> np.ndarray:
    t = np.array([s.as_tuple() for s in samples], dtype=np.float64).reshape(-1, 6)
    return np.ascontiguousarray(t.T) + 0.0


def _dev(torch, arr, dtype):
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device="cuda", dtype=dtype)


class DevicePlanner:
    """Stream-ordered device schedule for one graph/config, buffers sized for ``max_batch``.

    ``plan_tokens`` runs K1 (6-tuples from token counts) then K2-K4; ``plan_times``
    starts from given 6-tuples.  Results stay in HBM: ``orders[n_sec, B]`` with
    per-section rank offsets ``sec_off[n_sec, MAX_DP+1]``, critical-rank
    ``metrics[dp, 3]`` and ``evals[dp]``; ``err`` holds the error word.
    """

    def __init__(self, graph: SectionGraph, configs: Mapping[str, SectionConfig],
                 policy=ExecPolicy.INTERLEAVED, max_batch: int = N.MAX_BATCH, device=None):
        torch = _torch()
        self.torch = torch
        self.graph, self.configs = graph, dict(configs)
        self.policy = ExecPolicy.parse(policy)
        self.gs = N.graph_struct(graph, self.configs)
        self.tables = graph.tables
        n_sec = len(self.tables.section_ids)
        self.dp_crit = self.configs[graph.critical.id].dp
        self.max_batch = max_batch
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        i32 = dict(dtype=torch.int32, device=dev)
        self.times = torch.zeros(6 * max_batch, dtype=torch.float64, device=dev)
        self.ids = torch.zeros(max_batch, **i32)
        self.act = torch.zeros(max_batch, **i32)
        self.orders = torch.zeros(n_sec * max_batch, **i32)
        self.sec_off = torch.zeros(n_sec * (N.MAX_DP + 1), **i32)
        self.metrics = torch.zeros(3 * self.dp_crit, dtype=torch.float64, device=dev)
        self.evals = torch.zeros(self.dp_crit, dtype=torch.int64, device=dev)
        ws = N.lib().maestro_schedule_workspace(max_batch, self.dp_crit)
        self.work = torch.zeros((ws + 7) // 8, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int64, device=dev)
        self.B = 0

    # -- launches (no sync) -------------------------------------------------------
    def _check_b(self, B: int) -> None:
        if B <= 0:
            raise EmptyBatch("cannot schedule an empty batch")
        if B > self.max_batch:
            raise NativeError(f"batch {B} exceeds planner capacity {self.max_batch}")
        if -(-B // self.dp_crit) > N.MAX_RANK_SAMPLES:
            raise NativeError(f"more than {N.MAX_RANK_SAMPLES} samples on one critical rank")

    def plan_times(self, B: int, stream=None) -> None:
        """K2-K4 on ``self.times[:6B]`` (phase-major), ``self.ids``, ``self.act``."""
        self._check_b(B)
        self.B = B
        L, s = N.lib(), N.stream_ptr(stream)
        N.check(L.maestro_error_reset(N.ptr(self.err), s), "error_reset")
        N.check(L.maestro_build_schedule(ctypes_ref(self.gs), N.ptr(self.times), N.ptr(self.ids),
                                         N.ptr(self.act), B, self.policy.code, N.ptr(self.orders),
                                         N.ptr(self.sec_off), N.ptr(self.metrics), N.ptr(self.evals),
                                         N.ptr(self.work), N.ptr(self.err), s), "build_schedule")

    def plan_tokens(self, cost_table, tokens, B: int, stream=None) -> None:
        """K1 (+K2-K4): ``tokens`` int32 [n_bits, B] on device, ``cost_table`` f64 [n_bits, 8]."""
        self._check_b(B)
        self.B = B
        L, s = N.lib(), N.stream_ptr(stream)
        N.check(L.maestro_error_reset(N.ptr(self.err), s), "error_reset")
        N.check(L.maestro_sample_times(ctypes_ref(self.gs), N.ptr(cost_table), N.ptr(tokens), B,
                                       N.ptr(self.times), N.ptr(self.act), N.ptr(self.err), s), "sample_times")
        N.check(L.maestro_build_schedule(ctypes_ref(self.gs), N.ptr(self.times), N.ptr(self.ids),
                                         N.ptr(self.act), B, self.policy.code, N.ptr(self.orders),
                                         N.ptr(self.sec_off), N.ptr(self.metrics), N.ptr(self.evals),
                                         N.ptr(self.work), N.ptr(self.err), s), "build_schedule")

    def plan_tokens_graphed(self, cost_table, tokens, B: int, stream=None) -> None:
        """``plan_tokens`` replayed from a CUDA graph: the five launches (error reset, K1, K2, K3,
        K4) are captured once per (cost table, token buffer, B) and replayed as one graph launch
        -- the executors whose plan inputs live in fixed device buffers (KD) use it every step."""
        torch = self.torch
        key = (cost_table.data_ptr(), tokens.data_ptr(), int(B))
        if getattr(self, "_graph_key", None) != key:
            self._check_b(B)
            cap = torch.cuda.Stream(device=self.ids.device)
            cap.wait_stream(torch.cuda.current_stream(self.ids.device))
            with torch.cuda.stream(cap):
                self.plan_tokens(cost_table, tokens, B)  # warm-up: kernel attributes set outside capture
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                self.plan_tokens(cost_table, tokens, B)
            torch.cuda.current_stream(self.ids.device).wait_stream(cap)
            self._graph, self._graph_key = graph, key
        self.B = B
        if stream is None:
            self._graph.replay()
        else:
            with torch.cuda.stream(stream):
                self._graph.replay()

    # -- host readback (syncs) ----------------------------------------------------------
    def raise_errors(self, ids=None) -> None:
        N.raise_device_error(int(self.err.item()), ids, self.tables.section_ids)

    def host_orders(self) -> dict[tuple[int, int], np.ndarray]:
        """{(section index, rank): batch indices} for the critical and every auxiliary."""
        B = self.B
        orders = self.orders.cpu().numpy()
        off = self.sec_off.cpu().numpy().reshape(-1, N.MAX_DP + 1)
        out = {}
        t = self.tables
        for s in [t.critical, *t.merge_order]:
            dp = self.configs[t.section_ids[s]].dp
            for q in range(dp):
                out[(s, q)] = orders[s * B + off[s, q]: s * B + off[s, q + 1]].copy()
        return out


def ctypes_ref(gs):
    import ctypes

    return ctypes.byref(gs)


# ----------------------------------------------------------------------------- public API
def sort_initial(samples: Sequence[SampleTiming]) -> list[SampleTiming]:
    """Ascending t_f_bc, stable (scheduling.py:76-78)."""
    return sorted(samples, key=lambda s: s.t_f_bc)


def _single_rank(samples: Sequence[SampleTiming]):
    torch = _torch()
    B = len(samples)
    times = _dev(torch, _times_host(samples).reshape(-1), torch.float64)
    return torch, B, times


def rank_metrics(order: Sequence[SampleTiming], policy=ExecPolicy.INTERLEAVED) -> RankMetrics:
    """3-resource timeline of one rank (scheduling.py:81-152), evaluated on the device."""
    policy = ExecPolicy.parse(policy)
    if not order:
        return RankMetrics(0.0, 0.0, 0.0)
    torch, B, times = _single_rank(order)
    idx = torch.arange(B, dtype=torch.int32, device="cuda")
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    N.check(N.lib().maestro_rank_metrics(N.ptr(times), B, N.ptr(idx), B, policy.code, N.ptr(out),
                                         N.stream_ptr()), "rank_metrics")
    mk, busy, span = out.cpu().tolist()
    return RankMetrics(mk, busy, span)


def calculate_makespan(order: Sequence[SampleTiming], policy=ExecPolicy.INTERLEAVED) -> float:
    return rank_metrics(order, policy).makespan


def schedule_rank(samples: Sequence[SampleTiming], policy=ExecPolicy.INTERLEAVED,
                  counter: Optional[EvalCounter] = None) -> list[SampleTiming]:
    """Greedy best-position insertion (Alg. 1, scheduling.py:162-199) on the device."""
    policy = ExecPolicy.parse(policy)
    n = len(samples)
    if n <= 1:
        return list(samples)
    if n > N.MAX_RANK_SAMPLES:
        raise NativeError(f"more than {N.MAX_RANK_SAMPLES} samples on one rank")
    torch, B, times = _single_rank(samples)
    part = torch.arange(n, dtype=torch.int32, device="cuda")
    part_off = torch.tensor([0, n], dtype=torch.int32, device="cuda")
    orders = torch.zeros(n, dtype=torch.int32, device="cuda")
    metrics = torch.zeros(3, dtype=torch.float64, device="cuda")
    evals = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.check(N.lib().maestro_wavefront(N.ptr(times), B, N.ptr(part), N.ptr(part_off), 1, policy.code,
                                      N.ptr(orders), N.ptr(metrics), N.ptr(evals), N.stream_ptr()), "wavefront")
    if counter is not None:
        counter.count += int(evals.item())
    return [samples[i] for i in orders.cpu().tolist()]


def partition_batch(global_batch: Sequence[SampleTiming], dp_critical: int,
                    graph: Optional[SectionGraph] = None) -> dict[int, list[SampleTiming]]:
    """LPT partition across critical DP ranks (scheduling.py:202-264) on the device."""
    if not global_batch:
        raise EmptyBatch("cannot partition an empty batch")
    if dp_critical < 1:
        raise FanoutMismatch(f"dp_critical must be >= 1, got {dp_critical}")
    torch = _torch()
    if graph is None:
        graph = _sided_pseudo_graph()
    configs = {sid: SectionConfig() for sid in graph.section_ids}
    configs[graph.critical.id] = SectionConfig(dp=dp_critical)
    gs = N.graph_struct(graph, configs)
    B = len(global_batch)
    tab = graph.tables
    masks = np.array([tab.mask_of(s.activated_sections) if graph is not _PSEUDO else 0 for s in global_batch],
                     dtype=np.uint32)
    times = _dev(torch, _times_host(global_batch).reshape(-1), torch.float64)
    ids = _dev(torch, np.array([s.sample_id for s in global_batch]), torch.int32)
    act = _dev(torch, masks.view(np.int32), torch.int32)
    i32 = dict(dtype=torch.int32, device="cuda")
    up, down, lpt, part = (torch.zeros(B, **i32) for _ in range(4))
    part_off = torch.zeros(dp_critical + 1, **i32)
    err = torch.zeros(1, dtype=torch.int64, device="cuda")
    L, s = N.lib(), N.stream_ptr()
    N.check(L.maestro_error_reset(N.ptr(err), s), "error_reset")
    N.check(L.maestro_partition(ctypes_ref(gs), N.ptr(times), N.ptr(ids), N.ptr(act), B, N.ptr(up),
                                N.ptr(down), N.ptr(lpt), N.ptr(part), N.ptr(part_off), N.ptr(err), s), "partition")
    word = int(err.item())
    if word != N.ERR_CLEAN and ((word >> 24) & 0xFF) != 7:  # duplicate ids are build_schedule's check
        N.raise_device_error(word, [s.sample_id for s in global_batch])
    off = part_off.cpu().tolist()
    p = part.cpu().tolist()
    return {r: [global_batch[i] for i in p[off[r]: off[r + 1]]] for r in range(dp_critical)}


_PSEUDO = None


def _sided_pseudo_graph() -> SectionGraph:
    """graph=None keys aux load by side ("upstream"/"downstream", scheduling.py:231-236):
    a 3-section chain with one candidate per side auto-attributes exactly that way."""
    global _PSEUDO
    if _PSEUDO is None:
        from .workload import Edge, ExecMode, Role, SectionSpec, StructuralParams, build_graph

        st = StructuralParams(1, 1, 1, 1, 1)
        _PSEUDO = build_graph(
            [SectionSpec("upstream", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD, st),
             SectionSpec("critical", Role.CRITICAL, ExecMode.FORWARD_BACKWARD, st),
             SectionSpec("downstream", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD, st)],
            [Edge("upstream", "critical"), Edge("critical", "downstream")],
        )
    return _PSEUDO


def merge_fanout(rank_schedules: Sequence[Sequence[T]], fanout: int) -> list[T]:
    """Round-robin interleave of `fanout` rank orders (scheduling.py:267-285).

    Generic over Python objects, so it stays on the host; the device form is
    fused into K4 (csrc/plan.cu fanout_merge_kernel)."""
    if fanout < 1:
        raise FanoutMismatch(f"fanout must be >= 1, got {fanout}")
    if len(rank_schedules) != fanout:
        raise FanoutMismatch(f"expected {fanout} downstream rank schedules, got {len(rank_schedules)}")
    longest = max((len(r) for r in rank_schedules), default=0)
    return [r[i] for i in range(longest) for r in rank_schedules if i < len(r)]


def build_schedule(graph: SectionGraph, configs: Mapping[SectionId, SectionConfig],
                   batch: Sequence[SampleTiming], policy=ExecPolicy.INTERLEAVED) -> Schedule:
    """partition -> per-rank wavefront -> fan-out merge (scheduling.py:309-373), on the device."""
    policy = ExecPolicy.parse(policy)
    if not batch:
        raise EmptyBatch("cannot schedule an empty batch")
    planner = DevicePlanner(graph, configs, policy, max_batch=len(batch))
    B = len(batch)
    torch = planner.torch
    tab = planner.tables
    planner.times[: 6 * B].copy_(torch.from_numpy(_times_host(batch).reshape(-1)))
    ids = np.array([s.sample_id for s in batch], dtype=np.int32)
    planner.ids[:B].copy_(torch.from_numpy(ids))
    masks = np.array([tab.mask_of(s.activated_sections) for s in batch], dtype=np.uint32)
    planner.act[:B].copy_(torch.from_numpy(masks.view(np.int32)))
    planner.plan_times(B)
    planner.raise_errors(ids)
    per_rank = {(tab.section_ids[s], q): tuple(int(ids[i]) for i in o)
                for (s, q), o in planner.host_orders().items()}
    return Schedule(per_rank_orders=per_rank, batch=tuple(batch), policy=policy)


__all__ = [
    "ExecPolicy", "RankMetrics", "EvalCounter", "Schedule", "DevicePlanner", "sort_initial", "rank_metrics",
    "calculate_makespan", "schedule_rank", "partition_batch", "merge_fanout", "build_schedule", "PHASES",
]
