"""Generic section-graph executor: ``step()`` for any section graph, driven by the device schedule.

The execution contract is the reference executor model's stage queues (``maestro/simulator.py``
lines 202-233), at micro-batch granularity: every section rank hosted by this process is a
resource (a CUDA stream) that runs a fixed queue derived from the wavefront schedule --

* UPSTREAM sections: every forward micro-batch (f_bc) in schedule order, then every backward
  (b_ac) in the same order (none for forward-only sections);
* the CRITICAL section: per micro-batch forward then backward (``ExecPolicy.INTERLEAVED``) or all
  forwards then all backwards (``ALL_FWD_THEN_BWD``);
* DOWNSTREAM sections: f_ac / b_bc per critical micro-batch holding samples that activate them,
  in the same policy order;

and a stage starts once its resource is free and its chain predecessors (on other resources)
have finished: f_c(m) after the f_bc micro-batches holding m's samples, f_ac(m) after f_c(m),
b_c(m) after b_bc(m), b_ac(k) after the b_c micro-batches holding k's samples.  Dependencies are
CUDA events; the host enqueues stages in a topological order of that graph (an event must be
recorded before another stream waits on it).  Downstream micro-batches follow the critical
micro-batches (the samples of m that activate the section), so an interleaved critical queue can
never wait on a downstream micro-batch that needs a later critical forward.

Data between sections moves through per-step row buffers, placed by the K5b handoff indices
(``handoff.py``, computed on device from the schedule's orders) and the K6 row scatter:

* upstream -> critical "embed" edges: the encoder's output rows land at the sample's placeholder
  rows of the packed backbone stream (VLM / omni); gradients go back the same way;
* upstream -> critical "target" edges: the forward-only teacher's final hidden states, aligned
  with the student's tokens, feed the colocated teacher head and the fused KL loss (K9) (KD,
  workload.py:471-514);
* critical -> downstream edges: the backbone's final hidden rows of the sample's output span feed
  the downstream decoder; its input gradient is added into the backbone's final-hidden gradient.

With ``torch.distributed`` initialised every section is data-parallel over all ranks (the
co-located layout: each GPU hosts one rank of every section, fan-out 1) and each section's
gradients are summed over the group before its optimizer (C2; the loss scales use the global
batch's label / token counts, so the sum is the global gradient).  ``KDExecutor`` / ``VLMExecutor``
are the tuned special cases of this contract for cfg 2/5 and cfg 1 (plan-ahead, disjoint GPU
groups); ``tests/test_graph_exec.py`` checks that this executor reproduces their steps.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import dense as D
from . import kernels as K
from .costs import cost_table
from .errors import DependencyDeadlock
from .executor import StageClock, StepStats
from .handoff import HandoffIndex, handoff_index, scatter_mb
from .scheduling import DevicePlanner, ExecPolicy
from .transformer import Batch, FlatParams, Shape, Transformer
from .workload import Side


# --------------------------------------------------------------------------------------- inputs
@dataclass
class UpInput:
    """One upstream section's per-sample inputs (arrays over sample ids, length B)."""

    in_len: np.ndarray              # input rows per sample (patches / frames / tokens); 0 = not activated
    rows: np.ndarray                # rows handed to the critical section (in_len // merge)
    dst_off: np.ndarray             # placeholder offset of those rows inside the sample's sequence
    feats: np.ndarray | None = None  # [sum in_len, in_dim] fp32 rows in sample-id order (None: reads ids)


@dataclass
class DownInput:
    """One downstream section's per-sample inputs."""

    rows: np.ndarray                # backbone rows handed down per sample (0 = not activated)
    src_off: np.ndarray             # their offset inside the sample's sequence
    targets: np.ndarray             # [sum rows] int32 labels in sample-id order (decoder CE)


@dataclass
class GraphBatch:
    lens: np.ndarray                # critical sequence length per sample
    ids: np.ndarray                 # [B, Lmax] int32; -1 = placeholder (filled by an embed edge)
    labels: np.ndarray | None       # [B, Lmax] int32 next-token labels (-1 = none); None for KD
    up: dict = field(default_factory=dict)
    down: dict = field(default_factory=dict)
    _pinned: dict = field(default_factory=dict, repr=False)

    @property
    def B(self) -> int:
        return int(self.lens.shape[0])

    def pinned(self, key: str, arr: np.ndarray, bf16: bool = False) -> torch.Tensor:
        """Page-locked copy of an input array, built once per batch (a pinning loader's output);
        every step still copies it to the device."""
        hit = self._pinned.get(key)
        if hit is None or hit[0] is not arr:
            if bf16:
                x = np.ascontiguousarray(arr, dtype=np.float32).view(np.uint32)
                h = ((x + 0x7FFF + ((x >> 16) & 1)) >> 16).astype(np.uint16).view(np.int16)
                t = torch.from_numpy(h).pin_memory()
            else:
                t = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory()
            hit = (arr, t)
            self._pinned[key] = hit
        return hit[1]


# --------------------------------------------------------------------------------------- modules
class EncoderModule:
    """Upstream trainable encoder: input rows -> linear embed -> bidirectional stack -> 4:1 merge
    of consecutive rows (inputs arrive in merge-window order, as Qwen2.5-VL's patcher emits them)
    -> projector into the backbone width."""

    kind = "features"

    def __init__(self, shape: Shape, in_dim: int, out_d: int, merge: int, device, seed: int, max_pos: int = 16384):
        self.s, self.in_dim, self.out_d, self.merge = shape, in_dim, out_d, merge
        extra = [("in_w", (shape.d, in_dim)), ("proj_w", (out_d, merge * shape.d))]
        self.p = FlatParams(shape.param_shapes() + extra, device, trainable=True, seed=seed)
        self.model = Transformer(shape, self.p, device, max_pos=max_pos)
        self.device = device
        self.trainable = True

    def forward(self, x: torch.Tensor, cu: torch.Tensor, pos: torch.Tensor, max_len: int, out: torch.Tensor):
        x0 = D.linear_fwd(x, self.p["in_w"])
        yf, ctx = self.model.forward(Batch(ids=None, cu=cu, pos=pos, max_len=max_len), x0=x0)
        merged = yf.view(-1, self.merge * self.s.d)
        D.linear_fwd(merged, self.p["proj_w"], out)
        return dict(ctx=ctx, merged=merged, x=x)

    def backward(self, st, drows: torch.Tensor) -> None:
        D.linear_wgrad(drows, st["merged"], self.p.g("proj_w"))
        dyf = D.linear_dgrad(drows, self.p["proj_w"], wt=self.p.t("proj_w")).view(-1, self.s.d)
        dx0 = self.model.backward(st["ctx"], dyf=dyf, need_dx0=True)
        D.linear_wgrad(dx0, st["x"], self.p.g("in_w"))


class TeacherModule:
    """Upstream forward-only stack (KD teacher): token ids -> final hidden states (the teacher's
    output layer is colocated with the student, workload.colocate_output_layer)."""

    kind = "ids"

    def __init__(self, shape: Shape, device, seed: int, max_pos: int = 8192):
        self.s = shape
        self.p = FlatParams(shape.param_shapes(), device, trainable=False, seed=seed)
        self.model = Transformer(shape, self.p, device, max_pos=max_pos)
        self.trainable = False
        self.out_d = shape.d

    def forward(self, ids: torch.Tensor, cu: torch.Tensor, pos: torch.Tensor, max_len: int, out: torch.Tensor):
        self.model.forward(Batch(ids=ids, cu=cu, pos=pos, max_len=max_len), save=False, yf_out=out)
        return None


class DecoderModule:
    """Downstream trainable decoder: backbone rows -> projector -> causal stack -> head -> CE on
    its targets; returns the gradient of its input rows."""

    def __init__(self, shape: Shape, in_d: int, device, seed: int, max_pos: int = 8192):
        self.s, self.in_d = shape, in_d
        extra = [("in_w", (shape.d, in_d))]
        self.p = FlatParams(shape.param_shapes() + extra, device, trainable=True, seed=seed)
        self.model = Transformer(shape, self.p, device, max_pos=max_pos)
        self.device = device
        self.trainable = True

    def forward(self, x: torch.Tensor, cu: torch.Tensor, pos: torch.Tensor, max_len: int, targets: torch.Tensor,
                grad_scale: float, loss_acc: torch.Tensor):
        """f_ac: loss and d(logits) (kept in place of the logits for the backward)."""
        x0 = D.linear_fwd(x, self.p["in_w"])
        yf, ctx = self.model.forward(Batch(ids=None, cu=cu, pos=pos, max_len=max_len), x0=x0)
        logits = self.model.logits(yf)
        tl = torch.empty(x.shape[0], device=x.device)
        K.ce_loss(logits, targets, logits, tl, grad_scale)
        loss_acc.add_(tl.sum(), alpha=grad_scale)
        return dict(ctx=ctx, dlogits=logits, x=x)

    def backward(self, st, dx_out: torch.Tensor) -> None:
        """b_bc: parameter gradients and the gradient of the input rows (into dx_out)."""
        dx0 = self.model.backward(st["ctx"], dlogits=st["dlogits"], need_dx0=True)
        D.linear_wgrad(dx0, st["x"], self.p.g("in_w"))
        D.linear_dgrad(dx0, self.p["in_w"], out=dx_out, wt=self.p.t("in_w"))


class BackboneModule:
    """Critical section: decoder LM over the packed stream.  loss "ce": next-token cross entropy
    on the text labels (fused K9-family CE kernel); loss "kd": KL(teacher || student) over the full
    vocabulary with the teacher's colocated output layer (``t_head``) applied to the teacher rows."""

    def __init__(self, shape: Shape, device, seed: int, loss: str = "ce", t_head: torch.Tensor | None = None,
                 max_pos: int = 8192):
        self.s = shape
        self.p = FlatParams(shape.param_shapes(), device, trainable=True, seed=seed)
        self.model = Transformer(shape, self.p, device, max_pos=max_pos)
        self.loss, self.t_head = loss, t_head
        self.trainable = True


# --------------------------------------------------------------------------------------- executor
def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


@dataclass
class _Stage:
    res: str          # resource (section id)
    kind: str         # f_bc, b_ac, f_c, b_c, f_ac, b_bc
    m: int            # micro-batch index on its resource (critical index for f_ac / b_bc)
    deps: list        # [(res, kind, m)] chain predecessors on other resources


class SectionGraphExecutor:
    """``step(batch)`` over ``graph`` with ``modules[section_id]`` (EncoderModule / TeacherModule
    upstream, BackboneModule critical, DecoderModule downstream) and per-section ``configs``
    (``SectionConfig``: dp = world size, mbs = micro-batch samples)."""

    def __init__(self, graph, configs, modules, cost_params, policy=ExecPolicy.INTERLEAVED, device=None,
                 lr: float = 3e-4, max_batch: int = 1024, dp_group=None):
        self.graph, self.configs, self.mod = graph, dict(configs), dict(modules)
        self.policy = ExecPolicy.parse(policy)
        self.device = dev = device or torch.device("cuda", torch.cuda.current_device())
        tab = graph.tables
        self.tab = tab
        self.crit = tab.section_ids[tab.critical]
        self.ups = [s for s in tab.section_ids if graph.side(s) is Side.UPSTREAM]
        self.downs = [s for s in tab.section_ids if graph.side(s) is Side.DOWNSTREAM]
        dist = _dist()
        self.rank = dist.get_rank() if dist else 0
        self.world = dist.get_world_size() if dist else 1
        self.dp_group = dp_group
        for s, c in self.configs.items():
            if c.dp != self.world or c.fanout != 1:
                raise ValueError(f"section {s}: the co-located executor needs dp == world ({self.world}) and fanout 1")
        self.planner = DevicePlanner(graph, self.configs, self.policy, max_batch=max_batch, device=dev)
        self.cost = torch.from_numpy(cost_table(graph, self.configs, cost_params)).to(dev)
        self.streams = {s: torch.cuda.Stream(device=dev) for s in tab.section_ids}
        self.lr = lr
        self.step_idx = 0
        self._h_err = torch.empty(1, dtype=torch.int64).pin_memory()
        # C2 of the critical section overlapped with its last micro-batch's backward
        self.gsync = None
        import os

        if dist is not None and self.world > 1 and os.environ.get("MAESTRO_C2_OVERLAP", "1") != "0":
            from .gradsync import GradSync

            cm = self.mod[self.crit]
            self.gsync = GradSync(cm.p, cm.s.layers, group=dp_group, device=dev)

    # ---------------------------------------------------------------- planning (device, K1-K5)
    def _tokens(self, gb: GraphBatch) -> np.ndarray:
        tab, B = self.tab, gb.B
        tok = np.zeros((len(tab.sub_names), B), dtype=np.int32)
        per = {self.crit: gb.lens}
        for s in self.ups:
            per[s] = gb.up[s].in_len
        for s in self.downs:
            per[s] = gb.down[s].rows
        for bit, name in enumerate(tab.sub_names):
            owner = tab.section_ids[tab.sub_owner[bit]]
            if name == owner:
                tok[bit] = per[owner]
        return tok

    def _plan(self, gb: GraphBatch, stream) -> dict:
        dev, B = self.device, gb.B
        with torch.cuda.stream(stream):
            tokens = _h2d(self._tokens(gb), dev)
            self.planner.ids[:B].copy_(_h2d(np.arange(B, dtype=np.int32), dev))
            self.planner.plan_tokens(self.cost, tokens, B, stream)
            self._h_err.copy_(self.planner.err, non_blocking=True)
        orders = self.planner.host_orders()  # one small readback (synchronises)
        N.raise_device_error(int(self._h_err.item()), list(range(B)), self.tab.section_ids)
        idx = {s: i for i, s in enumerate(self.tab.section_ids)}
        return {s: orders[(idx[s], self.rank)].astype(np.int64) for s in self.tab.section_ids}

    # ---------------------------------------------------------------- one step
    def step(self, gb: GraphBatch, want_loss: bool = True) -> StepStats:
        """One iteration; programmatic dependent launch is off while it enqueues (the sections'
        streams run concurrently and early dependent CTAs would hold SMs the other streams use:
        cfg 3/4 measured -1 % with it, r02_pdl_section_ab.jsonl)."""
        prev = N.set_pdl(False)
        try:
            return self._step(gb, want_loss)
        finally:
            N.set_pdl(prev)

    def _step(self, gb: GraphBatch, want_loss: bool = True) -> StepStats:
        dev, B = self.device, gb.B
        main = torch.cuda.current_stream(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(main)
        orders = self._plan(gb, main)
        o_c = orders[self.crit]
        mbs_c = self.configs[self.crit].mbs
        z = lambda k: torch.empty(max(k, 1), dtype=torch.int32, device=dev)  # noqa: E731
        s = main.cuda_stream
        # ---- inputs (pinned host -> device) and the critical pack (K5)
        up_ = lambda key, a: gb.pinned(key, a).to(dev, non_blocking=True)  # noqa: E731
        lens = up_("lens32", gb.__dict__.setdefault("_lens32", gb.lens.astype(np.int32)))
        ids = up_("ids", gb.ids)
        labels = up_("labels", gb.labels) if gb.labels is not None else None
        n = len(o_c)
        n_mb = -(-n // mbs_c)
        o_c_d = _h2d(o_c.astype(np.int32), dev)
        c_tok = {k: z(x) for k, x in (("mb", n), ("tok_off", n), ("mb_tok", n_mb), ("cu", n_mb * (mbs_c + 1)),
                                       ("mb_start", n_mb))}
        N.check(N.lib().maestro_varlen_pack(N.ptr(o_c_d), n, N.ptr(lens), mbs_c, N.ptr(c_tok["mb"]),
                                            N.ptr(c_tok["tok_off"]), N.ptr(c_tok["mb_tok"]), N.ptr(c_tok["cu"]),
                                            N.ptr(c_tok["mb_start"]), s), "varlen_pack")
        total = int(gb.lens[o_c].sum())
        p_ids, p_lab = z(total), z(total)
        N.check(N.lib().maestro_pack_tokens(N.ptr(ids), ids.shape[1], N.ptr(o_c_d), N.ptr(lens),
                                            N.ptr(c_tok["tok_off"]), n, N.ptr(p_ids), s), "pack_tokens")
        if labels is not None:
            N.check(N.lib().maestro_pack_tokens(N.ptr(labels), labels.shape[1], N.ptr(o_c_d), N.ptr(lens),
                                                N.ptr(c_tok["tok_off"]), n, N.ptr(p_lab), s), "pack_tokens")
        c_lens = gb.lens[o_c]
        c_start = np.concatenate([[0], np.cumsum(c_lens)]).astype(np.int64)
        mb_c = [(m * mbs_c, min(n, (m + 1) * mbs_c)) for m in range(n_mb)]
        err = torch.full((1,), N.ERR_CLEAN, dtype=torch.int64, device=dev)
        # ---- upstream sections: packed inputs per micro-batch, output row buffers, edge indices
        up = {}
        d_c = self.mod[self.crit].s.d
        for sec in self.ups:
            ui, mod, o_u = gb.up[sec], self.mod[sec], orders[sec]
            mbs_u = self.configs[sec].mbs
            nu = len(o_u)
            rows_h = ui.rows.astype(np.int64)
            e = dict(order=o_u, mbs=mbs_u, n_mb=-(-nu // mbs_u) if nu else 0)
            e["row_start"] = np.concatenate([[0], np.cumsum(rows_h[o_u])]).astype(np.int64)
            e["in_start"] = np.concatenate([[0], np.cumsum(ui.in_len[o_u])]).astype(np.int64)
            width = mod.out_d
            e["buf"] = torch.empty(max(int(rows_h.sum()), 1), width, device=dev, dtype=torch.bfloat16)
            if mod.trainable:
                e["gbuf"] = torch.zeros_like(e["buf"])
            o_u_d = _h2d(o_u.astype(np.int32), dev)
            in_len_d = _h2d(ui.in_len.astype(np.int32), dev)
            e["pack"] = {k: z(x) for k, x in (("mb", nu), ("tok_off", nu), ("mb_tok", e["n_mb"]),
                                               ("cu", e["n_mb"] * (mbs_u + 1)), ("mb_start", e["n_mb"]))}
            if nu:
                N.check(N.lib().maestro_varlen_pack(N.ptr(o_u_d), nu, N.ptr(in_len_d), mbs_u, N.ptr(e["pack"]["mb"]),
                                                    N.ptr(e["pack"]["tok_off"]), N.ptr(e["pack"]["mb_tok"]),
                                                    N.ptr(e["pack"]["cu"]), N.ptr(e["pack"]["mb_start"]), s),
                        "varlen_pack")
            if mod.kind == "features":
                # device gather of each micro-batch's input rows out of the sample-id-ordered
                # feature block: a handoff index with the identity order as producer (K5b)
                act = np.nonzero(ui.in_len > 0)[0]
                e["feats"] = gb.pinned(f"feats:{sec}", ui.feats, bf16=True).to(dev, non_blocking=True).view(torch.bfloat16)
                mb_in = [int(ui.in_len[o_u[k * mbs_u:(k + 1) * mbs_u]].sum()) for k in range(e["n_mb"])]
                e["feat_ix"] = handoff_index(_h2d(act.astype(np.int32), dev), o_u_d, e["pack"]["tok_off"], mbs_u,
                                             in_len_d, _h2d(np.zeros(B, np.int32), dev), int(ui.in_len.sum()),
                                             max(mb_in or [1]), err)
            else:  # reads token ids (teacher): packed in its own order
                tt = int(ui.in_len[o_u].sum())
                e["ids"] = z(tt)
                if nu:
                    N.check(N.lib().maestro_pack_tokens(N.ptr(ids), ids.shape[1], N.ptr(o_u_d), N.ptr(in_len_d),
                                                        N.ptr(e["pack"]["tok_off"]), nu, N.ptr(e["ids"]), s),
                            "pack_tokens")
            mb_rows = [int(rows_h[o_c[a:b]].sum()) for a, b in mb_c]
            e["ix"] = handoff_index(o_u_d, o_c_d, c_tok["tok_off"], mbs_c, _h2d(ui.rows.astype(np.int32), dev),
                                    _h2d(ui.dst_off.astype(np.int32), dev), int(rows_h[o_c].sum()),
                                    max(mb_rows or [1]), err)
            e["mb_of"] = {int(i): k // mbs_u for k, i in enumerate(o_u)}
            up[sec] = e
        # ---- downstream sections: row buffers aligned with the critical micro-batches
        down = {}
        for sec in self.downs:
            di, o_d = gb.down[sec], orders[sec]
            rows_h = di.rows.astype(np.int64)
            if list(o_d) != [int(i) for i in o_c if rows_h[i] > 0]:
                raise DependencyDeadlock(f"downstream section '{sec}' order is not the critical order filtered",
                                         resources=(sec,))
            e = dict(order=o_d)
            tot = int(rows_h[o_d].sum())
            e["buf"] = torch.empty(max(tot, 1), d_c, device=dev, dtype=torch.bfloat16)
            e["gbuf"] = torch.empty_like(e["buf"])
            # rows of critical micro-batch m inside the buffer (d's order = critical order filtered)
            cum = np.concatenate([[0], np.cumsum(rows_h[o_c])]).astype(np.int64)
            e["mb_rows"] = [(int(cum[a]), int(cum[b])) for a, b in mb_c]
            mb_rows = [b - a for a, b in e["mb_rows"]]
            e["ix"] = handoff_index(_h2d(o_d.astype(np.int32), dev), o_c_d, c_tok["tok_off"], mbs_c,
                                    _h2d(di.rows.astype(np.int32), dev), _h2d(di.src_off.astype(np.int32), dev),
                                    tot, max(mb_rows or [1]), err)
            # decoder targets in the buffer's row order, cu_seqlens per critical micro-batch
            t_off = np.concatenate([[0], np.cumsum(rows_h)]).astype(np.int64)
            tgt = np.concatenate([di.targets[t_off[i]:t_off[i + 1]] for i in o_d]) if len(o_d) else np.zeros(1)
            e["targets"] = _h2d(tgt.astype(np.int32), dev)
            e["cu"], e["pos"], e["maxlen"] = [], [], []
            for a, b in mb_c:
                r = [int(rows_h[i]) for i in o_c[a:b] if rows_h[i] > 0]
                cu = np.concatenate([[0], np.cumsum(r)]).astype(np.int32)
                e["cu"].append(_h2d(cu, dev))
                e["pos"].append(_h2d(np.concatenate([np.arange(x) for x in r]).astype(np.int32), dev) if r else None)
                e["maxlen"].append(max(r) if r else 0)
            down[sec] = e
        ready = torch.cuda.Event()
        ready.record(main)
        # ---- loss scales (global over ranks: every rank sees the whole host batch)
        scales = {}
        crit_mod = self.mod[self.crit]
        if crit_mod.loss == "kd":
            scales["crit"] = 1.0 / float(gb.lens.sum())
        else:
            scales["crit"] = 1.0 / max(int((gb.labels >= 0).sum()), 1)
        for sec in self.downs:
            scales[sec] = 1.0 / max(int(gb.down[sec].rows.sum()), 1)
        loss_acc = torch.zeros(1, device=dev)
        for sec, mod in self.mod.items():
            if mod.trainable:
                mod.p.zero_grad()
        # ---- stage queues (simulator.py:202-233) and their chain dependencies
        stages = self._queues(orders, up, down, mb_c, gb)
        clocks = {r: StageClock() for r in stages}
        ev = {}
        for r in stages:
            self.streams[r].wait_event(ready)
        state = dict(ctx_c={}, ctx_u={sec: {} for sec in self.ups})
        ctx = dict(gb=gb, orders=orders, up=up, down=down, mb_c=mb_c, c_tok=c_tok, c_lens=c_lens, c_start=c_start,
                   p_ids=p_ids, p_lab=p_lab, scales=scales, loss_acc=loss_acc, state=state)
        head = {r: 0 for r in stages}
        left = sum(len(q) for q in stages.values())
        while left:
            progressed = False
            for r, q in stages.items():
                while head[r] < len(q) and all(d in ev for d in q[head[r]].deps):
                    st = q[head[r]]
                    stream = self.streams[r]
                    for d in st.deps:
                        stream.wait_event(ev[d])
                    with torch.cuda.stream(stream):
                        clocks[r].begin(stream, f"{st.kind}{st.m}")
                        self._run(st, ctx)
                        clocks[r].end(stream)
                        e = torch.cuda.Event()
                        e.record(stream)
                    ev[(r, st.kind, st.m)] = e
                    head[r] += 1
                    left -= 1
                    progressed = True
            if not progressed:
                blocked = tuple(r for r in stages if head[r] < len(stages[r]))
                raise DependencyDeadlock(f"no enqueueable stage; blocked resources: {blocked}", resources=blocked)
        # ---- per-section gradient all-reduce (C2, sum) and optimizers, on each section's stream
        dist = _dist()
        for sec, mod in self.mod.items():
            if not mod.trainable:
                continue
            stream = self.streams[sec]
            with torch.cuda.stream(stream):
                if dist is not None and self.world > 1:
                    # every rank scaled its loss by the GLOBAL label / token counts (all ranks see
                    # the whole host batch), so the global gradient is the sum over ranks
                    if sec == self.crit and self.gsync is not None:
                        self.gsync.finish(stream)  # per-layer buckets already in flight
                    else:
                        dist.all_reduce(mod.p.grad, group=self.dp_group)
                mod.p.adamw(self.lr)
        for r in self.streams.values():
            main.wait_stream(r)
        if dist is not None and self.world > 1:
            dist.all_reduce(loss_acc, group=self.dp_group)
        N.raise_device_error(int(err.item()), list(range(B)), self.tab.section_ids)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(main)
        t1.synchronize()
        self.step_idx += 1
        self.last_clocks = (t0, clocks)
        busy, span = clocks[self.crit].busy_span()
        loss = float(loss_acc.item()) if want_loss else None
        return StepStats(loss, t0.elapsed_time(t1), busy, span)

    # ---------------------------------------------------------------- queues
    def _queues(self, orders, up, down, mb_c, gb) -> dict:
        pol_il = self.policy is ExecPolicy.INTERLEAVED
        o_c = orders[self.crit]
        q = {}
        mb_of_c = {int(i): k // self.configs[self.crit].mbs for k, i in enumerate(o_c)}
        # upstream: all forwards, then all backwards
        for sec in self.ups:
            e, mod = up[sec], self.mod[sec]
            fw = [_Stage(sec, "f_bc", k, []) for k in range(e["n_mb"])]
            bw = []
            if mod.trainable:
                for k in range(e["n_mb"]):
                    crit_mbs = sorted({mb_of_c[int(i)] for i in e["order"][k * e["mbs"]:(k + 1) * e["mbs"]]})
                    bw.append(_Stage(sec, "b_ac", k, [(self.crit, "b_c", m) for m in crit_mbs]))
            q[sec] = fw + bw
        # critical
        fwd, bwd = [], []
        for m, (a, b) in enumerate(mb_c):
            deps = []
            for sec in self.ups:
                ks = sorted({up[sec]["mb_of"][int(i)] for i in o_c[a:b] if int(i) in up[sec]["mb_of"]})
                deps += [(sec, "f_bc", k) for k in ks]
            fwd.append(_Stage(self.crit, "f_c", m, deps))
            bdeps = [(sec, "b_bc", m) for sec in self.downs if down[sec]["mb_rows"][m][1] > down[sec]["mb_rows"][m][0]]
            bwd.append(_Stage(self.crit, "b_c", m, bdeps))
        q[self.crit] = [x for pair in zip(fwd, bwd) for x in pair] if pol_il else fwd + bwd
        # downstream: per critical micro-batch that holds its samples
        for sec in self.downs:
            ms = [m for m, (a, b) in enumerate(down[sec]["mb_rows"]) if b > a]
            f = [_Stage(sec, "f_ac", m, [(self.crit, "f_c", m)]) for m in ms]
            bb = [_Stage(sec, "b_bc", m, []) for m in ms]
            q[sec] = [x for pair in zip(f, bb) for x in pair] if pol_il else f + bb
        return q

    # ---------------------------------------------------------------- stage bodies
    def _run(self, st: _Stage, c) -> None:
        dev = self.device
        gb, up, down, state = c["gb"], c["up"], c["down"], c["state"]
        if st.kind == "f_bc":
            e, mod, k = up[st.res], self.mod[st.res], st.m
            o = e["order"][k * e["mbs"]:(k + 1) * e["mbs"]]
            ui = gb.up[st.res]
            T = int(ui.in_len[o].sum())
            cu = e["pack"]["cu"][k * (e["mbs"] + 1): k * (e["mbs"] + 1) + len(o) + 1]
            pos = torch.empty(T, dtype=torch.int32, device=dev)
            K.positions(cu, len(o), pos)
            r0, r1 = int(e["row_start"][k * e["mbs"]]), int(e["row_start"][k * e["mbs"] + len(o)])
            out = e["buf"][r0:r1]
            max_len = int(ui.in_len[o].max())
            if mod.kind == "features":
                x = torch.empty(T, mod.in_dim, device=dev, dtype=torch.bfloat16)
                scatter_mb(e["feat_ix"], k, e["feats"], x)
                state["ctx_u"][st.res][k] = mod.forward(x, cu, pos, max_len, out)
            else:
                i0 = int(e["in_start"][k * e["mbs"]])
                mod.forward(e["ids"][i0:i0 + T], cu, pos, max_len, out)
        elif st.kind == "b_ac":
            e, mod, k = up[st.res], self.mod[st.res], st.m
            n_k = len(e["order"][k * e["mbs"]:(k + 1) * e["mbs"]])
            r0, r1 = int(e["row_start"][k * e["mbs"]]), int(e["row_start"][k * e["mbs"] + n_k])
            mod.backward(state["ctx_u"][st.res].pop(k), e["gbuf"][r0:r1])
        elif st.kind == "f_c":
            self._crit_fwd(st.m, c)
        elif st.kind == "b_c":
            self._crit_bwd(st.m, c)
        elif st.kind == "f_ac":
            e, mod, m = down[st.res], self.mod[st.res], st.m
            a, b = e["mb_rows"][m]
            # critical rows -> this section's buffer (reverse direction of the index)
            scatter_mb(e["ix"], m, state["ctx_c"][m]["yf"], e["buf"], reverse=True)
            state.setdefault("ctx_d", {})[(st.res, m)] = mod.forward(
                e["buf"][a:b], e["cu"][m], e["pos"][m], e["maxlen"][m], e["targets"][a:b], c["scales"][st.res],
                c["loss_acc"])
        elif st.kind == "b_bc":
            e, mod, m = down[st.res], self.mod[st.res], st.m
            a, b = e["mb_rows"][m]
            mod.backward(state["ctx_d"].pop((st.res, m)), e["gbuf"][a:b])

    def _crit_fwd(self, m, c) -> None:
        dev, mod = self.device, self.mod[self.crit]
        a, b = c["mb_c"][m]
        mbs = self.configs[self.crit].mbs
        start, T = int(c["c_start"][a]), int(c["c_start"][b] - c["c_start"][a])
        cu = c["c_tok"]["cu"][m * (mbs + 1): m * (mbs + 1) + (b - a) + 1]
        pos = torch.empty(T, dtype=torch.int32, device=dev)
        K.positions(cu, b - a, pos)
        bt = Batch(ids=c["p_ids"][start: start + T], cu=cu, pos=pos, max_len=int(c["c_lens"][a:b].max()))
        d = mod.s.d
        x0 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
        K.embed(mod.p["embed"], bt.ids, x0)
        target = None
        for sec in self.ups:
            e, um = c["up"][sec], self.mod[sec]
            if um.kind == "features":  # embed edge: encoder rows at the placeholder rows
                scatter_mb(e["ix"], m, e["buf"], x0)
            else:  # target edge: teacher rows aligned with the student's tokens
                target = torch.empty(T, um.out_d, device=dev, dtype=torch.bfloat16)
                scatter_mb(e["ix"], m, e["buf"], target)
        yf, fctx = mod.model.forward(bt, x0=x0)
        logits = mod.model.logits(yf)
        tl = torch.empty(T, device=dev)
        if mod.loss == "kd":
            t_logits = torch.empty_like(logits)
            D.linear_fwd(target, mod.t_head, t_logits)  # colocated teacher output layer
            K.kd_loss(t_logits, logits, logits, tl, grad_scale=c["scales"]["crit"])
            del t_logits
        else:
            K.ce_loss(logits, c["p_lab"][start: start + T], logits, tl, c["scales"]["crit"])
        c["loss_acc"].add_(tl.sum(), alpha=c["scales"]["crit"])
        c["state"]["ctx_c"][m] = dict(ctx=fctx, logits=logits, yf=yf, ids=bt.ids)

    def _crit_bwd(self, m, c) -> None:
        mod = self.mod[self.crit]
        sc = c["state"]["ctx_c"].pop(m)

        def hook(dyf):
            for sec in self.downs:
                scatter_mb(c["down"][sec]["ix"], m, c["down"][sec]["gbuf"], dyf, accumulate=True)

        need_dx0 = any(self.mod[s].trainable and self.mod[s].kind == "features" for s in self.ups)
        layer_hook = None
        if self.gsync is not None and m == len(c["mb_c"]) - 1:  # the last b_c finalises every layer
            self.gsync.begin()
            layer_hook = self.gsync.layer_done
        dx0 = mod.model.backward(sc["ctx"], dlogits=sc["logits"], need_dx0=True, dyf_hook=hook if self.downs else None,
                                 layer_hook=layer_hook)
        K.embed_bwd(dx0, sc["ids"], mod.p.g("embed"))
        if need_dx0:
            for sec in self.ups:
                if self.mod[sec].trainable and self.mod[sec].kind == "features":
                    scatter_mb(c["up"][sec]["ix"], m, dx0, c["up"][sec]["gbuf"], reverse=True)

    # ---------------------------------------------------------------- accounting
    def stage_events(self):
        """Device stage timestamps of the last step (ms from its start): {resource: [(name, t0, t1)]}."""
        t0, clocks = self.last_clocks
        return {r: [(nm, t0.elapsed_time(a), t0.elapsed_time(b)) for nm, a, b in cl.marks] for r, cl in clocks.items()}


def _h2d(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)


def _h2d_bf16(a: np.ndarray, dev) -> torch.Tensor:
    """fp32 host rows -> bf16 device rows (round to nearest even on the host, pinned upload)."""
    x = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    h = ((x + 0x7FFF + ((x >> 16) & 1)) >> 16).astype(np.uint16)
    return torch.from_numpy(h.view(np.int16)).pin_memory().to(dev, non_blocking=True).view(torch.bfloat16)
