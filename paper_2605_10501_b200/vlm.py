"""VLM section graph (BASELINE cfg 1): ViT encoder (upstream) -> GPT backbone (critical).

The executor follows the reference stage-queue contract (simulator.py:202-233) with the
device wavefront schedule deciding both orders:

* the critical (LLM) rank runs its micro-batches (mbs consecutive samples of its K3 order)
  forward+backward, interleaved;
* the upstream (ViT) rank runs all forward micro-batches of its K4 fan-out-merged order, then
  all backward micro-batches in the same order;
* an LLM micro-batch forward waits only for the ViT micro-batches that produced its images
  (CUDA events; the wavefront order puts text-only samples first so the LLM starts at t=0),
  and a ViT backward micro-batch waits for the LLM backwards that produced its gradients.

Handoff (co-resident): ViT final hidden -> 2x2 patch merge (K6 row gather) -> projector GEMM ->
image-token rows scattered into the LLM's packed embedding stream at placeholder positions
(K6 scatter); the backward gathers the placeholder-row gradients back (K6) and runs the ViT
backward.  Loss: next-token cross entropy over text targets (fused full-vocab CE kernel).
"""

from __future__ import annotations


import numpy as np
import torch

from . import _native as N
from . import dense as D
from . import kernels as K
from . import recipes as R
from .costs import cost_table
from .executor import StageClock, StepStats, handoff_mode
from .handoff import handoff_index, scatter_mb
from .scheduling import DevicePlanner, ExecPolicy
from .synthetic import rand_int
from .transformer import SHAPES, Batch, FlatParams, Transformer

PATCH_DIM = 3 * 16 * 16  # pixels per 16x16 RGB patch
GRID = 14                 # 224 / 16


def merge_index() -> np.ndarray:
    """Row gather for the 2x2 merge: merged row (i*7+j), part k <- patch (2i+k//2)*14 + 2j+k%2."""
    out = np.empty(49 * 4, dtype=np.int32)
    for i in range(7):
        for j in range(7):
            for k in range(4):
                out[(i * 7 + j) * 4 + k] = (2 * i + k // 2) * GRID + 2 * j + k % 2
    return out


def vlm_host_batch(B: int, seed: int = 0, vocab: int = 32768, step: int = 0):
    """Synthetic inputs of one step: padded ids/labels [B, Lmax], lengths, image flags, pixels."""
    meta = R.vlm_tiny(1, B, seed).extra
    has_img, tl, off = meta["has_image"], meta["text_len"], meta["img_offset"]
    lens = tl + np.where(has_img, R.VIT_MERGED, 0)
    Lmax = int(lens.max())
    ids = np.full((B, Lmax), -1, dtype=np.int32)
    labels = np.full((B, Lmax), -1, dtype=np.int32)
    toks = rand_int(seed + 977 * step, 4, np.arange(B * 512), 0, vocab - 1).astype(np.int32).reshape(B, 512)
    for i in range(B):
        t = toks[i, : tl[i]]
        if has_img[i]:
            o = off[i]
            seq = np.concatenate([t[:o], np.full(R.VIT_MERGED, -1, np.int32), t[o:]])
        else:
            seq = t
        ids[i, : lens[i]] = seq
        nxt = np.concatenate([seq[1:], [-1]])
        lab = np.where((seq >= 0) & (nxt >= 0), nxt, -1)
        labels[i, : lens[i]] = lab
    n_img = int(has_img.sum())
    g = np.random.default_rng(seed + step)
    pixels = (g.standard_normal((n_img, 196, PATCH_DIM)) * 0.5).astype(np.float32)
    img_ordinal = np.full(B, -1, dtype=np.int32)
    img_ordinal[np.nonzero(has_img)[0]] = np.arange(n_img, dtype=np.int32)
    return dict(ids=ids, labels=labels, lens=lens.astype(np.int32), has_img=has_img, img_offset=off,
                pixels=pixels, img_ordinal=img_ordinal, n_labels=int((labels >= 0).sum()))


class ViTSection:
    """Patch embed -> bidirectional encoder -> final norm -> 2x2 merge -> projector."""

    def __init__(self, shape, llm_d: int, device, seed: int):
        self.s = shape
        extra = [("patch_w", (shape.d, PATCH_DIM)), ("proj_w", (llm_d, 4 * shape.d))]
        self.p = FlatParams(shape.param_shapes() + extra, device, trainable=True, seed=seed)
        self.model = Transformer(shape, self.p, device, max_pos=256)
        self.device = device
        self.merge = torch.from_numpy(merge_index()).to(device)
        self.llm_d = llm_d

    def forward(self, pixels_bf16: torch.Tensor, n_img: int):
        """pixels [n_img*196, 768] -> (image token embeddings [n_img*49, llm_d], ctx)."""
        dev, s = self.device, self.s
        T = n_img * 196
        x0 = D.linear_fwd(pixels_bf16, self.p["patch_w"])
        cu = torch.arange(0, T + 1, 196, dtype=torch.int32, device=dev)
        pos = torch.empty(T, dtype=torch.int32, device=dev)
        K.positions(cu, n_img, pos)
        yf, ctx = self.model.forward(Batch(ids=None, cu=cu, pos=pos, max_len=196), x0=x0)
        src = (self.merge[None, :] + 196 * torch.arange(n_img, device=dev, dtype=torch.int32)[:, None]).reshape(-1)
        merged = torch.empty(n_img * 196, s.d, device=dev, dtype=torch.bfloat16)
        K.scatter_rows(yf, merged, src, torch.arange(src.numel(), device=dev, dtype=torch.int32))
        merged = merged.view(n_img * 49, 4 * s.d)
        emb = D.linear_fwd(merged, self.p["proj_w"])
        return emb, dict(ctx=ctx, merged=merged, src=src, pixels=pixels_bf16, n_img=n_img)

    def backward(self, demb: torch.Tensor, st) -> None:
        dev, s = self.device, self.s
        D.linear_wgrad(demb, st["merged"], self.p.g("proj_w"))
        dmerged = D.linear_dgrad(demb, self.p["proj_w"], wt=self.p.t("proj_w")).view(-1, s.d)
        dyf = torch.empty_like(dmerged)
        # un-merge: a permutation, so the scatter with swapped indices is its own inverse
        K.scatter_rows(dmerged, dyf, torch.arange(st["src"].numel(), device=dev, dtype=torch.int32), st["src"])
        dx0 = self.model.backward(st["ctx"], dyf=dyf, need_dx0=True)
        D.linear_wgrad(dx0, st["pixels"], self.p.g("patch_w"))


class LazyStepStats:
    """StepStats of an enqueued step, evaluated on first access (synchronises on the step's end
    event then): ``loss``, ``step_ms``, ``critical_busy_ms``, ``critical_span_ms``, ``stall_frac``."""

    def __init__(self, t0, t1, clock, loss_acc, grad_scale):
        self._args = (t0, t1, clock, loss_acc, grad_scale)
        self._st = None

    def _eval(self) -> StepStats:
        if self._st is None:
            t0, t1, clock, loss_acc, grad_scale = self._args
            t1.synchronize()
            busy, span = clock.busy_span()
            loss = float(loss_acc.item()) * grad_scale if loss_acc is not None else None
            self._st = StepStats(loss, t0.elapsed_time(t1), busy, span)
        return self._st

    def __getattr__(self, name):
        return getattr(self._eval(), name)


class VLMExecutor:
    """Co-resident VLM step on one GPU (cfg 1 layout "1 GPU").  With ``dp_group`` (a
    torch.distributed group) every rank runs the co-resident step on its own batch and the ViT and
    LLM gradients are averaged over the group before the optimizer (both sections data-parallel
    on the same GPUs: the co-located layout at N > 1)."""

    def __init__(self, batch: int = 64, mbs_llm: int = 8, mbs_vit: int = 8, seed: int = 0, lr: float = 3e-4,
                 policy=ExecPolicy.INTERLEAVED, device=None, dp_group=None):
        self.device = dev = device or torch.device("cuda", torch.cuda.current_device())
        self.batch, self.mbs_llm, self.mbs_vit = batch, mbs_llm, mbs_vit
        self.rec = R.vlm_tiny(1, batch, seed)
        from .workload import SectionConfig

        self.configs = {"llm": SectionConfig(dp=1, mbs=mbs_llm), "vit": SectionConfig(dp=1, mbs=mbs_vit)}
        self.graph = self.rec.graph
        self.llm_shape = SHAPES["vlm_gpt2l"]
        self.vit_shape = SHAPES["vit_tiny"]
        self.llm = Transformer(self.llm_shape, FlatParams(self.llm_shape.param_shapes(), dev, True, seed + 10), dev,
                               max_pos=1024)
        self.vit = ViTSection(self.vit_shape, self.llm_shape.d, dev, seed + 11)
        self.planner = DevicePlanner(self.graph, self.configs, policy, max_batch=batch, device=dev)
        self.cost = torch.from_numpy(cost_table(self.graph, self.configs, self.rec.params)).to(dev)
        self.lr = lr
        self.dp_group = dp_group
        self.s_plan = torch.cuda.Stream(device=dev)
        W = N.MAX_DP + 1
        n_sec = len(self.graph.tables.section_ids)
        self._h_orders = torch.empty(n_sec * batch, dtype=torch.int32).pin_memory()
        self._h_off = torch.empty(n_sec * W, dtype=torch.int32).pin_memory()
        self._h_err = torch.empty(1, dtype=torch.int64).pin_memory()
        self._pending = None  # (host batch, readback event, live inputs) of a plan enqueued ahead
        self.s_llm = torch.cuda.Stream(device=dev)
        self.s_vit = torch.cuda.Stream(device=dev)
        self.step_idx = 0
        tab = self.graph.tables
        self.bits = {n: i for i, n in enumerate(tab.sub_names)}

    def _plan(self, hb: dict, stream):
        """Enqueue K1-K4 for host batch ``hb`` on ``stream`` plus an asynchronous readback of the
        rank orders into pinned host buffers; returns (event of the readback, live inputs)."""
        dev, B = self.device, self.batch
        tok = np.zeros((len(self.bits), B), dtype=np.int32)
        tok[self.bits["llm"]] = hb["lens"]
        tok[self.bits["vit"]] = np.where(hb["has_img"], R.VIT_PATCHES, 0)
        if not hasattr(self, "_tok_dev"):  # fixed token buffer: the plan is replayed from a CUDA graph
            self._tok_dev = torch.empty(tok.shape, dtype=torch.int32, device=dev)
        with torch.cuda.stream(stream):
            tokens = torch.from_numpy(tok).pin_memory()
            self._tok_dev.copy_(tokens, non_blocking=True)
            ids = torch.arange(B, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
            self.planner.ids[:B].copy_(ids)
            self.planner.plan_tokens_graphed(self.cost, self._tok_dev, B, stream)
            self._h_orders.copy_(self.planner.orders[: self._h_orders.numel()], non_blocking=True)
            self._h_off.copy_(self.planner.sec_off, non_blocking=True)
            self._h_err.copy_(self.planner.err, non_blocking=True)  # K1-K4 error word
            ev = torch.cuda.Event()
            ev.record(stream)
        return ev, (tokens, ids)

    def step(self, hb: dict, want_loss: bool = True, next_hb: dict | None = None) -> StepStats:
        """One iteration from a host batch (vlm_host_batch); inputs are copied in per step.
        ``next_hb`` (the following step's batch, e.g. from a prefetching loader) lets the step
        enqueue that batch's schedule on a side stream while its own kernels run, so the next
        step starts without a planning round trip (the scheduler overlaps the step)."""
        dev, B = self.device, self.batch
        main = torch.cuda.current_stream(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(main)
        pin = pinned_inputs(hb)
        ids = pin["ids"].to(dev, non_blocking=True)
        labels = pin["labels"].to(dev, non_blocking=True)
        lens = pin["lens"].to(dev, non_blocking=True)
        pixels = pin["pixels"].to(dev, non_blocking=True).view(torch.bfloat16)
        # ---- device plan: K1 6-tuples -> K2-K4 schedule (enqueued by the previous step when it
        # was given this batch; otherwise now, on the main stream)
        if self._pending is not None and self._pending[0] is hb:
            ev = self._pending[1]
        else:
            if self._pending is not None:
                # a plan for another batch is in flight on s_plan and writes the same planner and
                # pinned buffers: let it land before re-planning on the main stream
                self._pending[1].synchronize()
            ev, live = self._plan(hb, main)
        self._pending = None
        tab = self.graph.tables
        ci, vi = tab.critical, tab.section_ids.index("vit")
        W = N.MAX_DP + 1
        # one small readback: both rank orders (<= 2 x 64 ints) define the micro-batch plan
        ev.synchronize()
        err = int(self._h_err.item())
        if err != N.ERR_CLEAN:
            N.raise_device_error(err, list(range(B)), self.graph.tables.section_ids)
        orders = self._h_orders.numpy().reshape(-1, B)
        off = self._h_off.numpy().reshape(-1, W)
        o_llm = orders[ci, :B].copy()
        n_vit = int(off[vi, 1])
        o_vit = orders[vi, :n_vit].copy()
        # ---- K5 pack of the LLM order; token ids + labels in schedule order
        o_llm_d = _h2d(o_llm, dev)
        n_mb = -(-B // self.mbs_llm)
        z = lambda k: torch.empty(k, dtype=torch.int32, device=dev)  # noqa: E731
        mb, tok_off, mb_tok, cu, mb_start = z(B), z(B), z(n_mb), z(n_mb * (self.mbs_llm + 1)), z(n_mb)
        s = main.cuda_stream
        N.check(N.lib().maestro_varlen_pack(N.ptr(o_llm_d), B, N.ptr(lens), self.mbs_llm, N.ptr(mb), N.ptr(tok_off),
                                            N.ptr(mb_tok), N.ptr(cu), N.ptr(mb_start), s), "varlen_pack")
        lens_h = hb["lens"]
        total = int(lens_h.sum())
        p_ids, p_lab = z(total), z(total)
        for src, dst in ((ids, p_ids), (labels, p_lab)):
            N.check(N.lib().maestro_pack_tokens(N.ptr(src), src.shape[1], N.ptr(o_llm_d), N.ptr(lens), N.ptr(tok_off),
                                                B, N.ptr(dst), s), "pack_tokens")
        # host mirrors of the per-sample offsets (the orders are already on the host)
        toff_h = np.concatenate([[0], np.cumsum(lens_h[o_llm])[:-1]]).astype(np.int64)
        ordinal = hb["img_ordinal"]
        n_vmb = -(-n_vit // self.mbs_vit)
        # K5b on device: (ViT-buffer row, LLM micro-batch row) pairs of every image token -- the
        # ViT writes 49 merged rows per image in its own order, each lands at the sample's
        # placeholder offset inside its LLM micro-batch
        pin_idx = pinned_index_inputs(hb)
        ix = handoff_index(_h2d(o_vit.astype(np.int32), dev), o_llm_d, tok_off, self.mbs_llm,
                           pin_idx["rows"].to(dev, non_blocking=True), pin_idx["dst_off"].to(dev, non_blocking=True),
                           49 * max(n_vit, 1), 49 * min(self.mbs_llm, max(n_vit, 1)))
        ready = torch.cuda.Event()
        ready.record(main)
        clock = StageClock()
        loss_acc = torch.zeros(1, device=dev)
        grad_scale = 1.0 / max(hb["n_labels"], 1)
        self.llm.p.zero_grad()
        self.vit.p.zero_grad()
        emb_buf = torch.empty(max(n_vit, 1) * 49, self.llm_shape.d, device=dev, dtype=torch.bfloat16)
        demb_buf = torch.zeros_like(emb_buf)
        vit_slot = {int(i): k for k, i in enumerate(o_vit)}  # sample -> slot in ViT order (dependencies)
        # ---- ViT forward queue (upstream f_bc in merged order)
        vit_fwd_ev, vit_ctx = [], []
        self.s_vit.wait_event(ready)
        with torch.cuda.stream(self.s_vit):
            for k in range(n_vmb):
                samples = o_vit[k * self.mbs_vit: (k + 1) * self.mbs_vit]
                idx = _h2d(ordinal[samples].astype(np.int64), dev)
                px = pixels.index_select(0, idx).view(-1, PATCH_DIM)
                emb, st = self.vit.forward(px, len(samples))
                emb_buf[k * self.mbs_vit * 49: k * self.mbs_vit * 49 + emb.shape[0]].copy_(emb)
                vit_ctx.append(st)
                e = torch.cuda.Event()
                e.record(self.s_vit)
                vit_fwd_ev.append(e)
        # ---- LLM queue: per micro-batch fwd + bwd (critical, interleaved)
        llm_bwd_ev = []
        d = self.llm_shape.d
        self.s_llm.wait_event(ready)
        with torch.cuda.stream(self.s_llm):
            for m in range(n_mb):
                ks = list(range(m * self.mbs_llm, min(B, (m + 1) * self.mbs_llm)))
                samples = o_llm[ks]
                start = int(toff_h[ks[0]])
                T = int(lens_h[samples].sum())
                cu_m = cu[m * (self.mbs_llm + 1): m * (self.mbs_llm + 1) + len(ks) + 1]
                # dependencies: ViT micro-batches holding this micro-batch's images
                slots = [vit_slot[int(i)] for i in samples if hb["has_img"][i]]
                if slots:
                    self.s_llm.wait_event(vit_fwd_ev[max(slots) // self.mbs_vit])
                clock.begin(self.s_llm, f"llm{m}")
                pos = torch.empty(T, dtype=torch.int32, device=dev)
                K.positions(cu_m, len(ks), pos)
                b = Batch(ids=p_ids[start: start + T], cu=cu_m, pos=pos, max_len=int(lens_h[samples].max()))
                x0 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
                K.embed(self.llm.p["embed"], b.ids, x0)
                if slots:  # K6 over this micro-batch's pairs of the device index
                    scatter_mb(ix, m, emb_buf, x0)
                yf, ctx = self.llm.forward(b, x0=x0)
                logits = self.llm.logits(yf)
                tl = torch.empty(T, device=dev)
                K.ce_loss(logits, p_lab[start: start + T], logits, tl, grad_scale)
                loss_acc.add_(tl.sum())
                dx0 = self.llm.backward(ctx, dlogits=logits, need_dx0=True)
                K.embed_bwd(dx0, b.ids, self.llm.p.g("embed"))
                if slots:
                    # gradients of the placeholder rows back to the image-token slots (the same
                    # pairs, reverse direction)
                    scatter_mb(ix, m, dx0, demb_buf, reverse=True)
                clock.end(self.s_llm)
                e = torch.cuda.Event()
                e.record(self.s_llm)
                llm_bwd_ev.append(e)
        # ---- ViT backward queue (upstream b_ac, same order), after the LLM grads it needs
        llm_mb_of = {int(o_llm[k]): k // self.mbs_llm for k in range(B)}
        with torch.cuda.stream(self.s_vit):
            for k in range(n_vmb):
                samples = o_vit[k * self.mbs_vit: (k + 1) * self.mbs_vit]
                self.s_vit.wait_event(llm_bwd_ev[max(llm_mb_of[int(i)] for i in samples)])
                a = k * self.mbs_vit * 49
                self.vit.backward(demb_buf[a: a + len(samples) * 49], vit_ctx[k])
            if self.dp_group is None:
                self.vit.p.adamw(self.lr)
        if self.dp_group is None:
            with torch.cuda.stream(self.s_llm):
                self.llm.p.adamw(self.lr)
        if next_hb is not None:
            # the next batch's schedule runs beside this step's tail (the host copies above were
            # made before the planner buffers are rewritten)
            self.s_plan.wait_event(ev)
            self._pending = (next_hb, *self._plan(next_hb, self.s_plan))
        main.wait_stream(self.s_llm)
        main.wait_stream(self.s_vit)
        if self.dp_group is not None:
            # per-section gradient average over the data-parallel group (C2), then the optimizers
            dist = _dist()
            world = dist.get_world_size(self.dp_group)
            for p in (self.llm.p, self.vit.p):
                dist.all_reduce(p.grad, group=self.dp_group)
                p.grad.mul_(1.0 / world)
            dist.all_reduce(loss_acc, group=self.dp_group)
            loss_acc.mul_(1.0 / world)
            self.vit.p.adamw(self.lr)
            self.llm.p.adamw(self.lr)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(main)
        self.step_idx += 1
        # no host synchronisation here: the statistics (and the loss) are read on first access, so
        # the host can enqueue the next step while this one runs
        return LazyStepStats(t0, t1, clock, loss_acc if want_loss else None, grad_scale)

    def model_flops_per_step(self, hb) -> float:
        L = self.llm_shape
        toks = int(hb["lens"].sum())
        avg = float(np.mean(hb["lens"]))
        llm = 3.0 * toks * L.fwd_flops_per_token(int(avg), with_head=True)
        V = self.vit_shape
        n_img = int(hb["has_img"].sum())
        vit = 3.0 * n_img * (196 * (V.fwd_flops_per_token(196, with_head=False) + 2 * PATCH_DIM * V.d)
                             + 49 * 2 * 4 * V.d * L.d)
        return llm + vit


def pinned_inputs(hb: dict) -> dict:
    """The batch's step inputs in page-locked host memory, built once per host batch (what a
    pinning data loader hands over): token ids, labels, lengths and the image patches as bf16
    bits.  Every step still copies them to the device; a pageable float32 upload of the patches
    (19 MB at cfg 1) blocked the host for milliseconds per step.  The cache is rebuilt when the
    dict holds different arrays; arrays modified in place must drop ``hb["_pinned"]``."""
    pin = hb.get("_pinned")
    keys = ("ids", "labels", "lens", "pixels")
    if pin is not None and any(pin["_src"][k] is not hb[k] for k in keys):
        pin = None  # the dict now holds other arrays: rebuild (arrays mutated in place are not detected)
    if pin is None:
        px = np.ascontiguousarray(hb["pixels"], dtype=np.float32).view(np.uint32)
        # round-to-nearest-even fp32 -> bf16 bits (as torch's .to(torch.bfloat16) does)
        px16 = ((px + 0x7FFF + ((px >> 16) & 1)) >> 16).astype(np.uint16)
        pin = {k: torch.from_numpy(np.ascontiguousarray(hb[k])).pin_memory() for k in ("ids", "labels", "lens")}
        pin["pixels"] = torch.from_numpy(px16.view(np.int16)).pin_memory()
        pin["_src"] = {k: hb[k] for k in keys}
        hb["_pinned"] = pin
    return pin


def pinned_index_inputs(hb: dict) -> dict:
    """Per-sample handoff inputs of K5b in page-locked memory, built once per host batch: rows
    exchanged (49 merged image tokens, 0 for text-only samples) and their placeholder offset."""
    pin = hb.get("_pinned_idx")
    if pin is None or pin["_src"] is not hb["has_img"]:
        rows = np.where(hb["has_img"], 49, 0).astype(np.int32)
        off = np.where(hb["has_img"], hb["img_offset"], 0).astype(np.int32)
        pin = {"rows": torch.from_numpy(rows).pin_memory(), "dst_off": torch.from_numpy(off).pin_memory(),
               "_src": hb["has_img"]}
        hb["_pinned_idx"] = pin
    return pin


def _h2d(a: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device through pinned staging (a pageable upload would block the host on the
    stream and serialise enqueue with execution)."""
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


class VLMGroupExecutor:
    """VLM step with the sections on disjoint GPU groups (cfg 1 layouts 2 / 4 / 8 GPUs).

    Global ranks [0, dp_vit) host ViT ranks, [dp_vit, dp_vit + dp_llm) host LLM (critical)
    ranks; ViT rank q serves LLM ranks q*f .. q*f+f-1 (the fan-out map, scheduling.py:366-371).
    Every rank builds the same device schedule (K1-K4) from the same batch, so both ends of every
    handoff know its contents:

    * forward: after ViT micro-batch k, ViT rank q pushes to each LLM rank r the merged image
      tokens of the samples of k owned by r ([n*49, d_llm] bf16, mq.Channel over NCCL);
    * backward: after LLM micro-batch m, rank r pushes the placeholder-row gradients of m's image
      samples back to q; q runs all forwards, then all backwards in the same order (the upstream
      stage order of simulator.py:202-233), each backward once its gradients have arrived.

    Activations and gradients of a pair travel on two separate NCCL groups so that neither
    direction's point-to-point queue can block the other.  Per-section gradient all-reduce runs
    over each section's own DP group.  The batch is ``batch_per_llm_rank * dp_llm`` samples.
    """

    def __init__(self, n_gpus: int, batch_per_llm_rank: int = 64, mbs_llm: int = 8, mbs_vit: int = 8,
                 seed: int = 0, lr: float = 3e-4, policy=ExecPolicy.INTERLEAVED, device=None):
        from . import mq
        from .workload import SectionConfig

        dist = _dist()
        if dist is None or dist.get_world_size() != n_gpus or n_gpus < 2:
            raise ValueError("VLMGroupExecutor needs torch.distributed with world size == n_gpus >= 2")
        self.rank, self.world = dist.get_rank(), n_gpus
        self.device = dev = device or torch.device("cuda", torch.cuda.current_device())
        self.dp_llm, self.dp_vit, self.f = R.VLM_LAYOUTS[n_gpus]
        if self.dp_llm + self.dp_vit != n_gpus:
            raise ValueError(f"layout {R.VLM_LAYOUTS[n_gpus]} does not fill {n_gpus} GPUs")
        self.batch = batch_per_llm_rank * self.dp_llm
        # a ViT rank serves f LLM ranks: its micro-batches grow with the fan-out so its launch count
        # per step stays that of one LLM rank's images (ViT-tiny micro-batches are launch-bound;
        # with pp = 1 the per-sample 6-tuple, hence the schedule, does not depend on mbs)
        self.mbs_llm, self.mbs_vit = mbs_llm, mbs_vit * self.f
        self.rec = R.vlm_tiny(n_gpus, self.batch, seed)
        self.configs = {"llm": SectionConfig(dp=self.dp_llm, mbs=mbs_llm),
                        "vit": SectionConfig(dp=self.dp_vit, fanout=self.f, mbs=mbs_vit)}
        self.graph = self.rec.graph
        self.llm_shape, self.vit_shape = SHAPES["vlm_gpt2l"], SHAPES["vit_tiny"]
        self.role = "vit" if self.rank < self.dp_vit else "llm"
        self.q = self.rank if self.role == "vit" else None           # ViT section rank
        self.r = self.rank - self.dp_vit if self.role == "llm" else None  # LLM section rank
        self.seed, self.lr = seed, lr
        if self.role == "llm":
            self.llm = Transformer(self.llm_shape, FlatParams(self.llm_shape.param_shapes(), dev, True, seed + 10),
                                   dev, max_pos=1024)
        else:
            self.vit = ViTSection(self.vit_shape, self.llm_shape.d, dev, seed + 11)
        self.stream = torch.cuda.Stream(device=dev)
        if handoff_mode() == "nccl":
            N.reserve_sms_for_comm()  # NCCL handoff kernels run concurrently with the section compute
        self.planner = DevicePlanner(self.graph, self.configs, policy, max_batch=self.batch, device=dev)
        self.cost = torch.from_numpy(cost_table(self.graph, self.configs, self.rec.params)).to(dev)
        self.bits = {n: i for i, n in enumerate(self.graph.tables.sub_names)}
        # process groups (created collectively, same order on every rank)
        g_llm = dist.new_group(list(range(self.dp_vit, n_gpus)))
        g_vit = dist.new_group(list(range(self.dp_vit)))
        self.sec_group = g_llm if self.role == "llm" else g_vit
        self.chan_fwd, self.chan_bwd = {}, {}
        nvlink = handoff_mode() == "nvlink"
        # largest fragment of a pair: a ViT micro-batch's images forward, an LLM micro-batch's
        # image rows backward
        slot = max(self.mbs_vit, self.mbs_llm) * 49 * self.llm_shape.d * 2 + (1 << 16)

        def transport(peer, group, role):
            if nvlink:  # one-sided copy-engine puts into the receiver's slot ring (csrc/p2p.cu)
                return mq.PeerTransport(peer=peer, role=role, slot_bytes=slot, slots=16, group=group)
            return mq.DistTransport(peer=peer, group=group)

        for r in range(self.dp_llm):
            q = r // self.f
            a, b = q, self.dp_vit + r
            gf, gb = dist.new_group([a, b]), dist.new_group([a, b])
            if self.rank == a:
                self.chan_fwd[r] = mq.Channel((0, 0), (0, 0), transport(b, gf, "send"))
                self.chan_bwd[r] = mq.Channel((0, 0), (0, 0), transport(b, gb, "recv"))
            elif self.rank == b:
                self.chan_fwd[q] = mq.Channel((0, 0), (0, 0), transport(a, gf, "recv"))
                self.chan_bwd[q] = mq.Channel((0, 0), (0, 0), transport(a, gb, "send"))
        self._eps = {}
        self.step_idx = 0

    # ------------------------------------------------------------------ plan (host view)
    def _plan_async(self, hb, stream):
        """Enqueue K1-K4 for ``hb`` on ``stream`` and an asynchronous readback of the orders, the
        rank offsets and the error word into pinned host buffers; returns the readback event."""
        dev, B = self.device, self.batch
        tok = np.zeros((len(self.bits), B), dtype=np.int32)
        tok[self.bits["llm"]] = hb["lens"]
        tok[self.bits["vit"]] = np.where(hb["has_img"], R.VIT_PATCHES, 0)
        if not hasattr(self, "_h_orders"):
            n_sec = len(self.graph.tables.section_ids)
            self._h_orders = torch.empty(n_sec * B, dtype=torch.int32).pin_memory()
            self._h_off = torch.empty(n_sec * (N.MAX_DP + 1), dtype=torch.int32).pin_memory()
            self._h_err = torch.empty(1, dtype=torch.int64).pin_memory()
        if not hasattr(self, "_tok_dev"):  # fixed token buffer: the plan is replayed from a CUDA graph
            self._tok_dev = torch.empty(tok.shape, dtype=torch.int32, device=dev)
        with torch.cuda.stream(stream):
            self._tok_dev.copy_(_h2d(tok, dev))
            self.planner.ids[:B].copy_(_h2d(np.arange(B, dtype=np.int32), dev))
            self.planner.plan_tokens_graphed(self.cost, self._tok_dev, B, stream)
            self._h_orders.copy_(self.planner.orders[: self._h_orders.numel()], non_blocking=True)
            self._h_off.copy_(self.planner.sec_off, non_blocking=True)
            self._h_err.copy_(self.planner.err, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return ev

    def _orders(self, hb, main, next_hb=None):
        """Rank orders of ``hb``: from a plan enqueued ahead by the previous step (plan-ahead) or
        planned now; with ``next_hb`` the next batch's plan is enqueued on a side stream so it
        overlaps this step (the host reads it at the next step without a device round trip)."""
        B = self.batch
        pend, self._pending = getattr(self, "_pending", None), None
        if pend is not None and pend[0] is hb:
            ev = pend[1]
        else:
            if pend is not None:
                pend[1].synchronize()  # a plan for another batch still writes the same buffers
            ev = self._plan_async(hb, main)
        ev.synchronize()
        N.raise_device_error(int(self._h_err.item()), list(range(B)), self.graph.tables.section_ids)
        tab = self.graph.tables
        ci, vi = tab.critical, tab.section_ids.index("vit")
        W = N.MAX_DP + 1
        off = self._h_off.numpy().reshape(-1, W).copy()
        orders = self._h_orders.numpy().reshape(-1, B).copy()
        if next_hb is not None:
            if not hasattr(self, "s_plan"):
                self.s_plan = torch.cuda.Stream(device=self.device)
            self._pending = (next_hb, self._plan_async(next_hb, self.s_plan))
        llm = [orders[ci, off[ci, r]: off[ci, r + 1]] for r in range(self.dp_llm)]
        vit = [orders[vi, off[vi, q]: off[vi, q + 1]] for q in range(self.dp_vit)]
        return llm, vit

    def _endpoint(self, peer, direction, rows):
        from . import mq

        key = (peer, direction, rows)
        if key not in self._eps:
            lay = mq.ShardLayout((rows, self.llm_shape.d))
            ch = (self.chan_fwd if direction == "fwd" else self.chan_bwd)[peer]
            self._eps[key] = mq.Endpoint((0, 0), mq.plan_reshard(lay, lay), {(0, 0): ch}, torch.bfloat16)
        return self._eps[key]

    # ------------------------------------------------------------------ one step
    def step(self, hb: dict, want_loss: bool = True, next_hb: dict | None = None) -> StepStats:
        """One iteration; ``next_hb`` (the following step's batch) lets the step plan that batch on a
        side stream while its own kernels run (plan-ahead, as VLMExecutor.step)."""
        dist = _dist()
        dev = self.device
        main = torch.cuda.current_stream(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(main)
        llm_orders, vit_orders = self._orders(hb, main, next_hb)
        owner = np.full(self.batch, -1, dtype=np.int64)
        for r, o in enumerate(llm_orders):
            owner[o] = r
        has_img = hb["has_img"]
        grad_scale = 1.0 / max(hb["n_labels"], 1)
        ready = torch.cuda.Event()
        ready.record(main)
        self.stream.wait_event(ready)
        clock = StageClock()
        loss_acc = torch.zeros(1, device=dev)
        (self.vit.p if self.role == "vit" else self.llm.p).zero_grad()
        with torch.cuda.stream(self.stream):
            if self.role == "vit":
                self._vit_step(hb, vit_orders[self.q], llm_orders, owner, clock)
            else:
                self._llm_step(hb, llm_orders[self.r], vit_orders[self.r // self.f], owner, clock, loss_acc,
                               grad_scale)
            p = self.vit.p if self.role == "vit" else self.llm.p
            if dist.get_world_size(self.sec_group) > 1:
                dist.all_reduce(p.grad, group=self.sec_group)
            p.adamw(self.lr)
        main.wait_stream(self.stream)
        # loss: sum over the LLM ranks (the ViT ranks contribute 0), after the compute stream
        dist.all_reduce(loss_acc)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(main)
        self.step_idx += 1
        loss = float(loss_acc.item()) * grad_scale if want_loss else None
        t1.synchronize()
        for ep in self._eps.values():
            ep.verify()
        busy, span = clock.busy_span()
        self._last = (t0, clock)
        return StepStats(loss, t0.elapsed_time(t1), busy, span)

    def timeline(self):
        """Stage (name, start ms, end ms) of the last step on this rank, relative to its start."""
        t0, clock = self._last
        return [(n, t0.elapsed_time(a), t0.elapsed_time(b)) for n, a, b in clock.marks]

    def _vit_step(self, hb, order, llm_orders, owner, clock):
        from . import mq

        dev, d = self.device, self.llm_shape.d
        mbs = self.mbs_vit
        peers = [r for r in range(self.dp_llm) if r // self.f == self.q]
        ordinal = hb["img_ordinal"]
        n_mb = -(-len(order) // mbs)
        ctxs = []
        with torch.cuda.stream(self.stream):
            pixels_all = pinned_inputs(hb)["pixels"].to(dev, non_blocking=True).view(torch.bfloat16)
        for k in range(n_mb):
            samples = order[k * mbs: (k + 1) * mbs]
            with torch.cuda.stream(self.stream):
                px = pixels_all.index_select(0, _h2d(ordinal[samples].astype(np.int64), dev))
            clock.begin(self.stream, f"f_bc{k}")
            emb, st = self.vit.forward(px.view(-1, PATCH_DIM), len(samples))
            clock.end(self.stream)
            ctxs.append(st)
            emb = emb.view(len(samples), 49, d)
            for r in peers:  # this micro-batch's tokens for each LLM rank it serves
                sel = [j for j, s in enumerate(samples) if owner[s] == r]
                if not sel:
                    continue
                part = torch.empty(len(sel) * 49, d, device=dev, dtype=torch.bfloat16)
                src = np.concatenate([np.arange(49) + 49 * j for j in sel]).astype(np.int32)
                K.scatter_rows(emb.view(-1, d), part, _h2d(src, dev),
                               torch.arange(part.shape[0], dtype=torch.int32, device=dev))
                meta = mq.MessageMeta(tuple(part.shape), 2, "vit", (0, 0), int(samples[sel[0]]))
                self.chan_fwd[r].push(part, meta, donate=True)
        # gradient messages per LLM peer, in that rank's micro-batch order
        expect = {}
        for r in peers:
            o = llm_orders[r]
            for m in range(-(-len(o) // self.mbs_llm)):
                mb_s = [int(s) for s in o[m * self.mbs_llm: (m + 1) * self.mbs_llm] if hb["has_img"][s]]
                if mb_s:
                    expect.setdefault(r, []).append(mb_s)
        got = {}  # sample -> (tensor, row offset)
        pulled = {r: 0 for r in expect}
        for k in range(n_mb):
            samples = [int(s) for s in order[k * mbs: (k + 1) * mbs]]
            for s in samples:  # pull (in per-peer order) until every sample's rows are here
                r = int(owner[s])
                while s not in got:
                    mb_s = expect[r][pulled[r]]
                    t, _ = self._endpoint(r, "bwd", len(mb_s) * 49).pull(validate=False)
                    for j, x in enumerate(mb_s):
                        got[x] = (t, j * 49)
                    pulled[r] += 1
            demb = torch.empty(len(samples) * 49, d, device=dev, dtype=torch.bfloat16)
            by_msg = {}
            for j, s in enumerate(samples):
                t, o = got.pop(s)
                by_msg.setdefault(id(t), (t, [], []))
                by_msg[id(t)][1].append(np.arange(49) + o)
                by_msg[id(t)][2].append(np.arange(49) + 49 * j)
            for t, sr, dr in by_msg.values():  # K6 row scatter from each gradient message
                K.scatter_rows(t, demb, _h2d(np.concatenate(sr).astype(np.int32), dev),
                               _h2d(np.concatenate(dr).astype(np.int32), dev))
            clock.begin(self.stream, f"b_ac{k}")
            self.vit.backward(demb, ctxs[k])
            clock.end(self.stream)

    def _llm_step(self, hb, order, vit_order, owner, clock, loss_acc, grad_scale):
        from . import mq

        dev, d = self.device, self.llm_shape.d
        B = len(order)
        mbs = self.mbs_llm
        s = self.stream.cuda_stream
        lens_h = hb["lens"]
        o_d = _h2d(order.astype(np.int32), dev)
        pin = pinned_inputs(hb)
        lens = pin["lens"].to(dev, non_blocking=True)
        ids = pin["ids"].to(dev, non_blocking=True)
        labels = pin["labels"].to(dev, non_blocking=True)
        n_mb = -(-B // mbs)
        z = lambda k: torch.empty(k, dtype=torch.int32, device=dev)  # noqa: E731
        mb, tok_off, mb_tok, cu, mb_start = z(B), z(B), z(n_mb), z(n_mb * (mbs + 1)), z(n_mb)
        N.check(N.lib().maestro_varlen_pack(N.ptr(o_d), B, N.ptr(lens), mbs, N.ptr(mb), N.ptr(tok_off),
                                            N.ptr(mb_tok), N.ptr(cu), N.ptr(mb_start), s), "varlen_pack")
        total = int(lens_h[order].sum())
        p_ids, p_lab = z(total), z(total)
        for src, dst in ((ids, p_ids), (labels, p_lab)):
            N.check(N.lib().maestro_pack_tokens(N.ptr(src), src.shape[1], N.ptr(o_d), N.ptr(lens), N.ptr(tok_off),
                                                B, N.ptr(dst), s), "pack_tokens")
        toff_h = np.concatenate([[0], np.cumsum(lens_h[order])[:-1]]).astype(np.int64)
        # forward messages from the ViT rank: one per ViT micro-batch holding our images
        msgs = []
        for k in range(-(-len(vit_order) // self.mbs_vit)):
            mine = [int(x) for x in vit_order[k * self.mbs_vit: (k + 1) * self.mbs_vit] if owner[x] == self.r]
            if mine:
                msgs.append(mine)
        q = self.r // self.f
        got, pulled = {}, 0
        for m in range(n_mb):
            ks = list(range(m * mbs, min(B, (m + 1) * mbs)))
            samples = order[ks]
            img = [int(x) for x in samples if hb["has_img"][x]]
            for x in img:
                while x not in got:
                    mine = msgs[pulled]
                    t, _ = self._endpoint(q, "fwd", len(mine) * 49).pull(validate=False)
                    for j, y in enumerate(mine):
                        got[y] = (t, j * 49)
                    pulled += 1
            start, T = int(toff_h[ks[0]]), int(lens_h[samples].sum())
            cu_m = cu[m * (mbs + 1): m * (mbs + 1) + len(ks) + 1]
            clock.begin(self.stream, f"c{m}")
            pos = torch.empty(T, dtype=torch.int32, device=dev)
            K.positions(cu_m, len(ks), pos)
            b = Batch(ids=p_ids[start: start + T], cu=cu_m, pos=pos, max_len=int(lens_h[samples].max()))
            x0 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
            K.embed(self.llm.p["embed"], b.ids, x0)
            dst_rows, by_msg = [], {}
            for k, i in zip(ks, samples):
                if hb["has_img"][i]:
                    t, o = got.pop(int(i))
                    base = int(toff_h[k]) - start + int(hb["img_offset"][i])
                    dst_rows.append(base)
                    by_msg.setdefault(id(t), (t, [], []))
                    by_msg[id(t)][1].append(np.arange(49) + o)
                    by_msg[id(t)][2].append(np.arange(49) + base)
            for t, sr, dr in by_msg.values():  # K6 scatter into the packed stream at the placeholders
                K.scatter_rows(t, x0, _h2d(np.concatenate(sr).astype(np.int32), dev),
                               _h2d(np.concatenate(dr).astype(np.int32), dev))
            yf, ctx = self.llm.forward(b, x0=x0)
            logits = self.llm.logits(yf)
            tl = torch.empty(T, device=dev)
            K.ce_loss(logits, p_lab[start: start + T], logits, tl, grad_scale)
            loss_acc.add_(tl.sum())
            dx0 = self.llm.backward(ctx, dlogits=logits, need_dx0=True)
            K.embed_bwd(dx0, b.ids, self.llm.p.g("embed"))
            if dst_rows:  # placeholder-row gradients back to the ViT rank, in micro-batch order
                g = torch.empty(len(dst_rows) * 49, d, device=dev, dtype=torch.bfloat16)
                src = np.concatenate([np.arange(49) + b0 for b0 in dst_rows]).astype(np.int32)
                K.scatter_rows(dx0, g, _h2d(src, dev),
                               torch.arange(g.shape[0], dtype=torch.int32, device=dev))
                meta = mq.MessageMeta(tuple(g.shape), 2, "llm", (0, 0), int(img[0]))
                self.chan_bwd[q].push(g, meta, donate=True)
            clock.end(self.stream)

    def model_flops_per_step(self, hb) -> float:
        return VLMExecutor.model_flops_per_step(self, hb)
