"""Section-graph executor: ``step()`` runs one training iteration of a section graph.

The execution contract is the reference executor model (``maestro/simulator.py:202-233``):
every (section, DP rank) is a resource that runs a fixed stage queue derived from the
wavefront schedule --

* UPSTREAM sections: all forward stages (f_bc) in schedule order, then all backward (b_ac);
* CRITICAL / DOWNSTREAM sections: per micro-batch forward then backward (INTERLEAVED), or all
  forwards then all backwards (ALL_FWD_THEN_BWD);

and a stage may start once its resource is free and its chain predecessor (possibly on another
section) has finished.  Here a resource is a CUDA stream on the GPU that hosts the section rank;
a chain predecessor on the same GPU is a CUDA event, on another GPU an NCCL send/recv on the
fan-out map (``scheduling.py:366-371``).  Per-step work:

1. plan on device: K1 6-tuples from token counts, K2-K4 wavefront schedule, K5 varlen pack of the
   local rank's order into micro-batches (one small D2H of micro-batch sizes per step);
2. run the local stage queues; stage boundaries are CUDA events, so the critical section's
   busy time and span -- the reference's ``critical_idle`` / section stall (scheduling.py:64-66,
   simulator.py:312-315) -- are measured on the device;
3. per-section gradient all-reduce over that section's own DP group, then the fused optimizer.

The KD graph (cfg 2) is implemented by :class:`KDExecutor`: a forward-only teacher upstream of
the student, with the teacher's output layer colocated in the student section
(``workload.colocate_output_layer``), so the teacher ships final hidden states ``[T, d_t]``
and the student computes teacher logits next to the fused KL loss (K9).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from . import recipes as R
from .costs import cost_table
from .scheduling import DevicePlanner, ExecPolicy
from .transformer import SHAPES, Batch, FlatParams, Shape, Transformer


@dataclass
class StepStats:
    loss: float | None
    step_ms: float
    critical_busy_ms: float
    critical_span_ms: float
    stages: list = field(default_factory=list)
    plan_ms: float = 0.0          # device time of the step's schedule build (K1-K5 + pack tables)
    allreduce_ms: float = 0.0     # student gradient all-reduce (C2), 0 at dp1
    teacher_busy_ms: float = 0.0  # summed teacher stage time on this rank (0 if not hosted)

    @property
    def stall_frac(self) -> float:
        return 0.0 if self.critical_span_ms <= 0 else max(0.0, 1.0 - self.critical_busy_ms / self.critical_span_ms)


class LazyKDStats:
    """StepStats of an enqueued KDExecutor step, evaluated on first attribute access (it then
    synchronises on the step's end event, reads the loss and checks the step's handoff headers)."""

    def __init__(self, ex, t0, t1, clock, t_clock, plan_t, ar, loss_acc, global_tokens, n_msgs):
        self._args = (ex, t0, t1, clock, t_clock, plan_t, ar, loss_acc, global_tokens, n_msgs)
        self._st = None

    def _eval(self) -> StepStats:
        if self._st is None:
            ex, t0, t1, clock, t_clock, plan_t, ar, loss_acc, global_tokens, n_msgs = self._args
            t1.synchronize()
            if n_msgs is not None:
                want, taken = n_msgs
                got = sorted(m.sample_id for ep, d in taken for m in ep.verify(d))  # this step's headers
                if got != list(range(want)):
                    from .errors import InconsistentSchedule

                    raise InconsistentSchedule("handoff delivered unexpected micro-batches", got=got)
            loss = float(loss_acc.item()) / global_tokens if loss_acc is not None else None
            busy, span = clock.busy_span()
            extra = {"plan_ms": plan_t[0].elapsed_time(plan_t[1]),
                     "teacher_busy_ms": t_clock.busy_span()[0] if ex.teacher is not None else 0.0}
            if ex.student is not None and ar is not None:
                extra["allreduce_ms"] = ar[0].elapsed_time(ar[1])
            self._st = StepStats(loss, t0.elapsed_time(t1), busy, span, **extra)
            self._args = (ex, None, None, None, None, None, None, None, None, None)
        return self._st

    def __getattr__(self, name):
        return getattr(self._eval(), name)


class StageClock:
    """CUDA events around every stage of one resource (stream)."""

    def __init__(self):
        self.marks = []

    def begin(self, stream, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.marks.append([name, e, None])

    def end(self, stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.marks[-1][2] = e

    def busy_span(self):
        if not self.marks:
            return 0.0, 0.0
        busy = sum(a.elapsed_time(b) for _, a, b in self.marks)
        span = self.marks[0][1].elapsed_time(self.marks[-1][2])
        return busy, span


def rank_roles(rank: int, n_gpus: int, layout: str = "colocated"):
    """Host-only placement of the KD section ranks (no device needed).

    Returns dict(t_rank, s_rank, dp_s, dp_t, colocated, send_to, recv_from, student_ranks):
    the teacher DP rank / student DP rank hosted by ``rank`` (None if absent), and the NCCL
    peer of the teacher->student handoff on the fan-out map (scheduling.py:366-371): teacher
    rank q serves student ranks q*f .. q*f+f-1; with fan-out 1 that is student rank q.
    """
    dp_s, dp_t, f, colocated = R.kd_layout(n_gpus, layout)
    if colocated:
        return dict(t_rank=rank, s_rank=rank, dp_s=dp_s, dp_t=dp_t, colocated=True, send_to=[], recv_from=[],
                    student_ranks=list(range(n_gpus)))
    t_rank = rank if rank < dp_t else None
    s_rank = rank - dp_t if rank >= dp_t else None
    send_to = [dp_t + q for q in range(t_rank * f, (t_rank + 1) * f)] if t_rank is not None else []
    recv_from = [s_rank // f] if s_rank is not None else []
    return dict(t_rank=t_rank, s_rank=s_rank, dp_s=dp_s, dp_t=dp_t, colocated=False, send_to=send_to,
                recv_from=recv_from, student_ranks=list(range(dp_t, n_gpus)))


def handoff_mode() -> str:
    """Cross-GPU handoff transport: "nvlink" (default; mq.PeerTransport, copy-engine puts and
    stream memory ops, no SMs) or "nccl" (mq.DistTransport, NCCL point-to-point)."""
    import os

    mode = os.environ.get("MAESTRO_HANDOFF", "nvlink")
    if mode not in ("nvlink", "nccl"):
        raise ValueError(f"MAESTRO_HANDOFF must be nvlink or nccl, got {mode!r}")
    return mode


def _prio_section() -> str:
    """MAESTRO_STREAM_PRIORITY=teacher|student|none: which co-resident section's stream gets the
    higher CUDA scheduling priority (its CTAs dispatched first when both have work).  Measured on
    cfg 2: student first -3 %, teacher first -0.7 % (r02_stream_priority_ab.jsonl); default none."""
    return os.environ.get("MAESTRO_STREAM_PRIORITY", "none")


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


class KDExecutor:
    """KD section graph (recipes.kd): teacher (upstream, forward-only) -> student (critical)."""

    def __init__(self, n_gpus: int = 1, batch_per_rank: int = 64, seq: int = R.KD_SEQ, mbs: int = 4,
                 teacher: str = "kd_teacher_1b", student: str = "kd_student_125m", seed: int = 0,
                 lr: float = 3e-4, policy=ExecPolicy.INTERLEAVED, device=None, layout: str = "colocated",
                 teacher_mbs: int | None = None, recipe: str = "kd"):
        dist = _dist()
        self.rank = dist.get_rank() if dist else 0
        self.world = dist.get_world_size() if dist else 1
        if self.world != n_gpus:
            raise ValueError(f"n_gpus={n_gpus} but world size is {self.world}")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.n_gpus, self.seq, self.mbs = n_gpus, seq, mbs
        # per-section micro-batch sizes (SectionConfig.mbs): the forward-only teacher may run larger
        # micro-batches (fuller last GEMM waves, fewer launches); a student micro-batch then reads
        # its rows out of the teacher micro-batch holding it (same sample order at fan-out 1)
        self.mbs_t = teacher_mbs or mbs
        if self.mbs_t % mbs:
            raise ValueError(f"teacher_mbs {self.mbs_t} must be a multiple of the student mbs {mbs}")
        self.mbs_of = {"student": mbs, "teacher": self.mbs_t}
        dp_s, dp_t, f_t, colocated = R.kd_layout(n_gpus, layout)
        self.layout = "colocated" if colocated else "disjoint"
        self.batch = batch_per_rank * dp_s
        # cfg 2 (recipes.kd) or cfg 5 (recipes.kd_8b): same graph shape, different cost knobs
        self.recipe = (R.kd_8b if recipe == "kd_8b" else R.kd)(n_gpus, self.batch, seq, self.layout)
        cfg = {"student": self.recipe.configs["student"].__class__(dp=dp_s, mbs=mbs),
               "teacher": self.recipe.configs["teacher"].__class__(dp=dp_t, fanout=f_t, mbs=self.mbs_t)}
        self.configs = cfg
        self.graph = self.recipe.graph
        # roles: co-resident teacher+student DP rank per GPU, or disjoint groups (teacher first)
        self.colocated = colocated
        self.roles = rank_roles(self.rank, n_gpus, self.layout)
        self.t_rank, self.s_rank = self.roles["t_rank"], self.roles["s_rank"]
        self.dp_s, self.dp_t = dp_s, dp_t
        self.tshape: Shape = SHAPES[teacher]
        self.sshape: Shape = SHAPES[student]
        dev = self.device
        # --- sections hosted here
        self.teacher = self.student = None
        if self.t_rank is not None:
            tp = FlatParams(self.tshape.param_shapes(), dev, trainable=False, seed=seed + 1)
            self.teacher = Transformer(self.tshape, tp, dev, max_pos=seq)
            self.t_stream = torch.cuda.Stream(device=dev, priority=-1 if _prio_section() == "teacher" else 0)
        if self.s_rank is not None:
            sp = FlatParams(self.sshape.param_shapes(), dev, trainable=True, seed=seed + 2)
            self.student = Transformer(self.sshape, sp, dev, max_pos=seq)
            # colocated teacher output layer (workload.colocate_output_layer): frozen, lives here
            g = torch.Generator(device=dev).manual_seed(seed + 3)
            self.t_head = (torch.randn(self.tshape.vocab, self.tshape.d, device=dev, generator=g) * 0.02).bfloat16()
            self.s_stream = torch.cuda.Stream(device=dev, priority=-1 if _prio_section() == "student" else 0)
        self.lr = lr
        # --- device planner (every rank computes the same deterministic schedule)
        self.planner = DevicePlanner(self.graph, cfg, policy, max_batch=self.batch, device=dev)
        self.cost = torch.from_numpy(cost_table(self.graph, cfg, self.recipe.params)).to(dev)
        tab = self.graph.tables
        self.n_bits = len(tab.sub_names)
        self._bits = {n: i for i, n in enumerate(tab.sub_names)}
        self.lens = torch.full((self.batch,), seq, dtype=torch.int32, device=dev)
        self.tokens = torch.zeros(self.n_bits, self.batch, dtype=torch.int32, device=dev)
        self.tokens[self._bits["student"]] = seq
        self.tokens[self._bits["teacher"]] = seq
        self.planner.ids[: self.batch].copy_(torch.arange(self.batch, dtype=torch.int32))
        self.groups = self._make_groups()
        # C2 overlapped with the last student micro-batch's backward (gradsync.GradSync)
        self.gsync = None
        if _dist() is not None and self.student is not None and dp_s > 1 and os.environ.get(
                "MAESTRO_C2_OVERLAP", "1") != "0":
            from .gradsync import GradSync

            self.gsync = GradSync(self.student.p, self.sshape.layers, group=self.groups.get("student"), device=dev)
        if not colocated and handoff_mode() == "nccl":
            N.reserve_sms_for_comm()  # NCCL handoff kernels run concurrently with the section compute
        self.step_idx = 0

    # ------------------------------------------------------------------ distributed plumbing
    def _make_groups(self):
        dist = _dist()
        if dist is None:
            return {}
        if self.colocated:  # student DP group = every rank
            return {"student": None, "student_ranks": list(range(self.world))}
        dp_t = self.dp_t
        s_ranks = list(range(dp_t, self.world))
        grp = dist.new_group(s_ranks) if len(s_ranks) > 1 else None
        return {"student": grp, "student_ranks": s_ranks}

    # ------------------------------------------------------------------ planning
    def plan(self, stream):
        """K1-K5 on device for this step; returns per-local-rank micro-batch tables (host)."""
        with torch.cuda.stream(stream):
            self.planner.plan_tokens_graphed(self.cost, self.tokens, self.batch, stream)
        tab = self.graph.tables
        crit, teach = tab.critical, tab.section_ids.index("teacher")
        out = {}
        W = N.MAX_DP + 1
        for sec, rank in (("student", self.s_rank), ("teacher", self.t_rank)):
            if rank is None:
                continue
            s = crit if sec == "student" else teach
            # orders of section s live at orders[s*B + off] (device); build the pack tables
            n_per = self.batch // (self.dp_s if sec == "student" else self.dp_t)
            off = self.planner.sec_off.view(-1, W)[s, rank: rank + 1]
            base = s * self.batch
            with torch.cuda.stream(stream):
                order = torch.empty(n_per, dtype=torch.int32, device=self.device)
                # device-side gather of the rank's slice (offset read on device via index_select)
                idx = (torch.arange(n_per, device=self.device, dtype=torch.int32) + off.to(torch.int32) + base).long()
                order.copy_(self.planner.orders.index_select(0, idx))
                mbs = self.mbs_of[sec]
                n_mb = -(-n_per // mbs)
                z = lambda k: torch.empty(k, dtype=torch.int32, device=self.device)  # noqa: E731
                mb, tok_off, mb_tok, cu, mb_start = z(n_per), z(n_per), z(n_mb), z(n_mb * (mbs + 1)), z(n_mb)
                N.check(N.lib().maestro_varlen_pack(N.ptr(order), n_per, N.ptr(self.lens), mbs, N.ptr(mb),
                                                    N.ptr(tok_off), N.ptr(mb_tok), N.ptr(cu), N.ptr(mb_start),
                                                    stream.cuda_stream), "varlen_pack")
            out[sec] = dict(order=order, tok_off=tok_off, mb_tok=mb_tok, cu=cu, mb_start=mb_start, n=n_per,
                            n_mb=n_mb, mbs=mbs)
        return out

    def serialized(self):
        """Context: co-resident sections share one stream (teacher micro-batches, then student
        ones) -- used to time each kernel without the other section's kernels sharing the GPU."""
        from contextlib import contextmanager

        @contextmanager
        def ctx():
            if not (self.colocated and self.teacher is not None and self.student is not None):
                yield self  # one section per rank: nothing to serialise
                return
            saved = self.s_stream
            self.s_stream = self.t_stream
            try:
                yield self
            finally:
                self.s_stream = saved

        return ctx()

    # ------------------------------------------------------------------ one step
    def _plan_async(self, stream):
        """K1-K5 for one step on ``stream`` plus an asynchronous readback of the micro-batch token
        counts into pinned host buffers; returns (tables, host buffers, readback event, device
        time events of the plan)."""
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        plan = self.plan(stream)
        p1.record(stream)
        bufs = {}
        with torch.cuda.stream(stream):
            for k, v in plan.items():
                a = torch.empty(v["n_mb"], dtype=torch.int32).pin_memory()
                b = torch.empty(v["n_mb"], dtype=torch.int32).pin_memory()
                a.copy_(v["mb_tok"], non_blocking=True)
                b.copy_(v["mb_start"], non_blocking=True)
                bufs[k] = (a, b)
            # the K1-K4 device error word travels with the readback: an invalid batch raises the
            # reference's exception class before any micro-batch is built (scheduling.py:217-365)
            err = torch.empty(1, dtype=torch.int64).pin_memory()
            err.copy_(self.planner.err, non_blocking=True)
            bufs["_err"] = err
            ev = torch.cuda.Event()
            ev.record(stream)
        return plan, bufs, ev, (p0, p1)

    def step(self, ids: torch.Tensor, want_loss: bool = True, plan_ahead: bool = False) -> StepStats:
        """One training iteration.  ``ids``: [batch, seq] int32 token ids (device or pinned host).
        ``plan_ahead``: after enqueueing this step, build the next step's schedule on a side stream
        so it overlaps this step (the sequence lengths -- the schedule's only input -- are fixed
        per executor), and the next step starts without a planning round trip."""
        dev = self.device
        main = torch.cuda.current_stream(dev)
        if ids.device.type != "cuda":
            ids_dev = torch.empty(ids.shape, dtype=torch.int32, device=dev)
            ids_dev.copy_(ids, non_blocking=True)
        else:
            ids_dev = ids
        t_start = torch.cuda.Event(enable_timing=True)
        t_start.record(main)
        pending, self._pending = getattr(self, "_pending", None), None
        plan, bufs, plan_ev, plan_t = pending if pending is not None else self._plan_async(main)
        # one small readback per step: micro-batch token counts of the local rank orders
        plan_ev.synchronize()
        main.wait_event(plan_ev)
        err = int(bufs["_err"].item())
        if err != N.ERR_CLEAN:
            N.raise_device_error(err, self.planner.ids[: self.batch].tolist(), self.graph.tables.section_ids)
        host = {k: (v[0].tolist(), v[1].tolist()) for k, v in bufs.items() if k != "_err"}
        packed = {}
        with torch.cuda.stream(main):
            for sec, v in plan.items():
                total = int(sum(host[sec][0]))
                pk = torch.empty(total, dtype=torch.int32, device=dev)
                N.check(N.lib().maestro_pack_tokens(N.ptr(ids_dev), ids_dev.shape[1], N.ptr(v["order"]),
                                                    N.ptr(self.lens), N.ptr(v["tok_off"]), v["n"], N.ptr(pk),
                                                    main.cuda_stream), "pack_tokens")
                packed[sec] = pk
        ready = torch.cuda.Event()
        ready.record(main)
        clock = StageClock()
        self.t_clock = StageClock()
        self.s_clock, self.t_origin = clock, t_start
        loss_acc = None
        if self.student is not None:
            loss_acc = torch.zeros(1, device=dev, dtype=torch.float32)
            self.student.p.zero_grad()
        global_tokens = float(self.batch * self.seq)
        if self.colocated:
            self._run_colocated(plan, host, packed, ready, clock, loss_acc, global_tokens)
        elif self.t_rank is not None:
            self._run_teacher_remote(plan, host, packed, ready)
        else:
            self._run_student_remote(plan, host, packed, ready, clock, loss_acc, global_tokens)
        # per-section gradient sync (student DP group) + optimizer, on the student stream
        ar = None  # (all-reduce start, end) events; none on a teacher-only rank
        if self.student is not None:
            with torch.cuda.stream(self.s_stream):
                dist = _dist()
                if dist is not None and self.dp_s > 1:
                    ar = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ar[0].record(self.s_stream)
                    if self.gsync is not None:  # per-layer buckets already in flight: the tail only
                        self.gsync.finish(self.s_stream)
                    else:
                        dist.all_reduce(self.student.p.grad, group=self.groups.get("student"))
                    dist.all_reduce(loss_acc, group=self.groups.get("student"))
                    ar[1].record(self.s_stream)
                self.student.p.adamw(self.lr)
            main.wait_stream(self.s_stream)
        if self.teacher is not None and not self.colocated:
            main.wait_stream(self.t_stream)
        if plan_ahead:
            if not hasattr(self, "s_plan"):
                self.s_plan = torch.cuda.Stream(device=dev)
            self.s_plan.wait_event(plan_ev)  # this step's plan has consumed the planner buffers
            self._pending = self._plan_async(self.s_plan)
        t_end = torch.cuda.Event(enable_timing=True)
        t_end.record(main)
        self.step_idx += 1
        # No end-of-step host synchronisation: the statistics (loss, stall, timings) and the
        # deferred handoff-header check are evaluated on first access, and at the latest when the
        # NEXT step has been enqueued -- so the host stays one step ahead of the device.
        n_msgs = None
        if self.student is not None and not self.colocated:  # this step's handoff headers, checked lazily
            n_msgs = (-(-plan["student"]["n_mb"] // (self.mbs_t // self.mbs)),
                      [(ep, ep.take_deferred()) for ep in getattr(self, "_h_eps", {}).values()])
        stats = LazyKDStats(self, t_start, t_end, clock, self.t_clock, plan_t, ar,
                            loss_acc if want_loss else None, global_tokens, n_msgs)
        prev, self._unchecked = getattr(self, "_unchecked", None), stats
        if prev is not None:
            prev._eval()
        return stats

    # --- co-resident sections on one GPU: the teacher stream runs ahead (upstream queue),
    # the student stream waits per micro-batch on a CUDA event.
    def _teacher_mb(self, packed, cu, m, start, T):
        b = Batch(ids=packed[start: start + T], cu=cu, pos=self._positions(cu, T), max_len=self.seq)
        yf, _ = self.teacher.forward(b, save=False)
        return yf

    def _positions(self, cu, T):
        pos = torch.empty(T, dtype=torch.int32, device=self.device)
        K.positions(cu, cu.numel() - 1, pos)
        return pos

    def _student_mb(self, yf_t, packed, cu, start, T, loss_acc, global_tokens, clock, m, last=False):
        b = Batch(ids=packed[start: start + T], cu=cu, pos=self._positions(cu, T), max_len=self.seq)
        clock.begin(self.s_stream, f"f_c{m}")
        yf, ctx = self.student.forward(b)
        s_logits = self.student.logits(yf)
        t_logits = torch.empty_like(s_logits)
        from . import dense as D

        D.linear_fwd(yf_t, self.t_head, t_logits)  # colocated teacher output layer
        tok_loss = torch.empty(T, device=self.device, dtype=torch.float32)
        K.kd_loss(t_logits, s_logits, s_logits, tok_loss, grad_scale=1.0 / global_tokens)
        loss_acc.add_(tok_loss.sum())
        del t_logits
        clock.end(self.s_stream)
        clock.begin(self.s_stream, f"b_c{m}")
        hook = None
        if last and self.gsync is not None:  # this backward finalises every layer's gradient
            self.gsync.begin()
            hook = self.gsync.layer_done
        self.student.backward(ctx, dlogits=s_logits, layer_hook=hook)
        clock.end(self.s_stream)

    def _mb_cu(self, plan_sec, m, T):
        mbs = plan_sec["mbs"]
        n_in = min(mbs, plan_sec["n"] - m * mbs)
        cu = plan_sec["cu"][m * (mbs + 1): m * (mbs + 1) + n_in + 1]
        return cu

    def _run_colocated(self, plan, host, packed, ready, clock, loss_acc, global_tokens):
        ps, pt = plan["student"], plan["teacher"]
        ht, hs = host["teacher"], host["student"]
        ev = []
        self.t_stream.wait_event(ready)
        self.s_stream.wait_event(ready)
        outs = []
        with torch.cuda.stream(self.t_stream):
            for m in range(pt["n_mb"]):
                T = ht[0][m]
                self.t_clock.begin(self.t_stream, f"f_bc{m}")
                yf = self._teacher_mb(packed["teacher"], self._mb_cu(pt, m, T), m, ht[1][m], T)
                self.t_clock.end(self.t_stream)
                e = torch.cuda.Event()
                e.record(self.t_stream)
                ev.append(e)
                outs.append(yf)
        ratio = self.mbs_t // self.mbs
        with torch.cuda.stream(self.s_stream):
            for m in range(ps["n_mb"]):
                # fan-out 1, same sample order: student micro-batch m's rows sit in teacher micro-batch
                # m // ratio at the token offset of its first sample
                k = m // ratio
                self.s_stream.wait_event(ev[k])
                T = hs[0][m]
                o = hs[1][m] - ht[1][k]
                self._student_mb(outs[k][o: o + T], packed["student"], self._mb_cu(ps, m, T), hs[1][m], T, loss_acc,
                                 global_tokens, clock, m, last=m == ps["n_mb"] - 1)
                if m % ratio == ratio - 1 or m == ps["n_mb"] - 1:
                    outs[k].record_stream(self.s_stream)
                    outs[k] = None

    # --- disjoint groups: the handoff (C1) is the reshard message queue (mq.py) over NCCL
    # point-to-point: the teacher rank pushes each micro-batch's final hidden state [T, d_t]
    # (identity layout: DP-only build, so plan_reshard yields one transfer per pair), the student
    # rank pulls it on its stream; headers are verified once per step (Endpoint.verify).
    def _handoff_channel(self, peer: int) -> "mq.Channel":
        from . import mq

        ch = getattr(self, "_h_chan", None)
        if ch is None:
            if handoff_mode() == "nvlink":  # one-sided copy-engine puts into the student's slot ring
                role = "send" if self.teacher is not None else "recv"
                slot = self.mbs_t * self.seq * self.tshape.d * 2 + (1 << 20)
                tr = mq.PeerTransport(peer=peer, role=role, slot_bytes=slot, slots=4 if slot > (64 << 20) else 8)
            else:
                tr = mq.DistTransport(peer=peer)
            ch = self._h_chan = mq.Channel((0, 0), (0, 0), tr)
        return ch

    def _handoff_endpoint(self, peer: int, T: int):
        from . import mq

        eps = self.__dict__.setdefault("_h_eps", {})
        if T not in eps:
            lay = mq.ShardLayout((T, self.tshape.d))
            eps[T] = mq.Endpoint((0, 0), mq.plan_reshard(lay, lay), {(0, 0): self._handoff_channel(peer)},
                                 torch.bfloat16)
        return eps[T]

    def _run_teacher_remote(self, plan, host, packed, ready):
        from . import mq

        pt, ht = plan["teacher"], host["teacher"]
        (dst,) = self.roles["send_to"]  # fan-out 1: teacher rank q feeds student rank q
        ch = self._handoff_channel(dst)
        self.t_stream.wait_event(ready)
        with torch.cuda.stream(self.t_stream):
            for m in range(pt["n_mb"]):
                T = ht[0][m]
                self.t_clock.begin(self.t_stream, f"f_bc{m}")
                yf = self._teacher_mb(packed["teacher"], self._mb_cu(pt, m, T), m, ht[1][m], T)
                self.t_clock.end(self.t_stream)
                meta = mq.MessageMeta((T, self.tshape.d), 2, "teacher", (0, 0), m)
                ch.push(yf, meta, donate=True)  # fresh buffer per micro-batch: no staging copy

    def _run_student_remote(self, plan, host, packed, ready, clock, loss_acc, global_tokens):
        ps, hs = plan["student"], host["student"]
        (src,) = self.roles["recv_from"]  # teacher rank feeding this student rank
        self.s_stream.wait_event(ready)
        with torch.cuda.stream(self.s_stream):
            ratio = self.mbs_t // self.mbs
            cur, cur_start = None, 0
            for m in range(ps["n_mb"]):
                T = hs[0][m]
                if m % ratio == 0:  # the teacher micro-batch holding this and the next ratio-1 ones
                    ms = list(range(m, min(ps["n_mb"], m + ratio)))
                    Tt = sum(hs[0][x] for x in ms)
                    cur, _ = self._handoff_endpoint(src, Tt).pull(validate=False)
                    cur_start = hs[1][m]
                o = hs[1][m] - cur_start
                self._student_mb(cur[o: o + T], packed["student"], self._mb_cu(ps, m, T), hs[1][m], T, loss_acc,
                                 global_tokens, clock, m, last=m == ps["n_mb"] - 1)

    def verify_handoff(self):
        """Check the deferred control headers of this step's pulls (sample ids in schedule order)."""
        got = []
        for ep in getattr(self, "_h_eps", {}).values():
            got += [m.sample_id for m in ep.verify()]
        return got

    # ------------------------------------------------------------------ measured timeline
    def measured_events(self):
        """Device stage timestamps of the last step as simulator StageEvents (sample id = micro-batch)."""
        from .simulator import measured_events

        if getattr(self, "_unchecked", None) is not None:
            self._unchecked._eval()  # the last step has completed (its events are readable)

        ev = []
        if self.teacher is not None and getattr(self, "t_clock", None) is not None:
            tev = measured_events(self.t_clock.marks, self.t_origin, "teacher", self.t_rank, lambda n: "f_bc")
            ratio = self.mbs_t // self.mbs
            if ratio > 1:  # a teacher micro-batch feeds `ratio` student micro-batches: one sub-stage each
                from dataclasses import replace

                split = []
                for e in tev:
                    d = (e.end - e.start) / ratio
                    split += [replace(e, sample_id=e.sample_id * ratio + i, start=e.start + i * d,
                                      end=e.start + (i + 1) * d) for i in range(ratio)]
                tev = split
            ev += tev
        if self.student is not None:
            ev += measured_events(self.s_clock.marks, self.t_origin, "student", self.s_rank,
                                  lambda n: "f_c" if n.startswith("f_c") else "b_c")
        return sorted(ev, key=lambda e: (e.start, e.section, e.dp_rank, e.sample_id, e.phase))

    def crosscheck(self):
        """Re-run the executor model (simulator.simulate) with the measured per-micro-batch stage
        durations; returns (modelled makespan s, modelled critical idle s, measured span s, measured
        critical idle s).  Co-resident sections share one GPU, so the model (one resource per
        section) bounds what a disjoint placement of the same stages would achieve."""
        from .scheduling import Schedule
        from .simulator import simulate
        from .workload import SampleTiming

        ev = self.measured_events()
        dur: dict = {}
        for e in ev:
            dur.setdefault(e.sample_id, {})[e.phase] = e.end - e.start
        batch = [SampleTiming(m, t_f_bc=d.get("f_bc", 0.0), t_f_c=max(d.get("f_c", 0.0), 1e-12),
                              t_b_c=d.get("b_c", 0.0), activated_sections=frozenset({"teacher"}))
                 for m, d in sorted(dur.items())]
        order = tuple(m for m, _ in sorted(dur.items()))
        from .workload import SectionConfig

        sched = Schedule(per_rank_orders={("student", 0): order, ("teacher", 0): order}, batch=tuple(batch))
        rep, _ = simulate(self.graph, {"student": SectionConfig(), "teacher": SectionConfig()}, sched)
        crit = [e for e in ev if e.section == "student"]
        span = crit[-1].end - crit[0].start if crit else 0.0
        busy = sum(e.end - e.start for e in crit)
        return rep.makespan, rep.critical_idle, span, span - busy

    # ------------------------------------------------------------------ accounting
    def attention_flops_per_step(self) -> tuple[float, float]:
        """Algorithmic attention FLOPs of one step over the whole job: (forward launches, backward
        launches) -- forward = teacher + student, 4*H*dh*L^2/2 per causal sequence per layer;
        backward = 2.5x the student's forward."""
        L = self.seq
        per = lambda s: s.layers * 4.0 * s.heads * s.head_dim * L * L * 0.5  # noqa: E731
        fwd = self.batch * (per(self.tshape) + per(self.sshape))
        return fwd, self.batch * 2.5 * per(self.sshape)

    def kd_loss_bytes_per_step(self) -> float:
        """Algorithmic bytes of K9 per step: read teacher + student logits, write dlogits (bf16)."""
        return self.batch * self.seq * self.tshape.vocab * 2.0 * 3

    def readback_bytes_per_step(self) -> int:
        """D2H bytes of one step on a student rank: the plan readback (micro-batch token counts and
        starts, int32, per hosted section) + the 8-byte error word + the fp32 loss."""
        n = 0
        for sec, rank in (("student", self.s_rank), ("teacher", self.t_rank)):
            if rank is not None:
                per = self.batch // (self.dp_s if sec == "student" else self.dp_t)
                n += 2 * 4 * (-(-per // self.mbs_of[sec]))
        return n + 8 + 4

    def model_flops_per_step(self) -> float:
        """Algorithmic FLOPs of one step over the whole job (teacher fwd + head, student train)."""
        s, t, L = self.sshape, self.tshape, self.seq
        tok = self.batch * L
        t_fwd = t.fwd_flops_per_token(L, with_head=True)  # teacher body + colocated head
        s_train = 3.0 * s.fwd_flops_per_token(L, with_head=True)
        return tok * (t_fwd + s_train)


def synthetic_ids(batch: int, seq: int, vocab: int, seed: int = 0, step: int = 0) -> np.ndarray:
    from .synthetic import rand_int

    n = batch * seq
    return rand_int(seed, 4 + 16 * step, np.arange(n), 0, vocab - 1).astype(np.int32).reshape(batch, seq)


def smoke_step():
    """Tiny KD step on cuda:0 (used by __graft_entry__.smoke)."""
    ex = KDExecutor(n_gpus=1, batch_per_rank=4, seq=256, mbs=2, teacher="test_tiny", student="test_tiny")
    ids = torch.from_numpy(synthetic_ids(4, 256, 512)).cuda()
    st = ex.step(ids)
    assert st.loss is not None and math.isfinite(st.loss), st
    st2 = ex.step(ids)
    assert math.isfinite(st2.loss)
    print(f"smoke kd step: loss {st.loss:.4f} -> {st2.loss:.4f}, stall {st.stall_frac:.3f}")
