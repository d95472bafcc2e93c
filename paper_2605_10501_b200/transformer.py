"""Section compute: Llama-style decoder blocks with explicit forward / backward on our kernels.

No autograd and no torch compute ops on the hot path: every FLOP goes through the tcgen05
GEMM (dense.py), the attention kernels (attention.py) or the memory-bound kernels
(kernels.py).  torch only allocates buffers and owns streams.

A block is   y1 = rmsnorm(h1) ; qkv = y1 Wqkv^T ; rope ; o = attn(qkv)
             h2 = h1 + o Wo^T ; y2 = rmsnorm(h2) ; gu = y2 Wgu^T ; s = silu(g) u ; h1' = h2 + s Wd^T
(Wgu stores gate/up rows interleaved in 32-row blocks so SwiGLU runs in the GEMM epilogue;
RoPE likewise runs in the QKV GEMM epilogue, and both residual adds in the epilogues of the
Wo / Wd projections, so the norms read the residual stream once.)  Parameters of a section live in one
flat arena (fp32 master, bf16 working copy, fp32 grad, Adam m/v) so the optimizer and the
gradient all-reduce are single launches over contiguous memory.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import attention as A
from . import dense as D
from . import kernels as K


@dataclass(frozen=True)
class Shape:
    d: int
    layers: int
    heads: int
    kv_heads: int
    ffn: int
    vocab: int
    head_dim: int = 64
    tied: bool = False
    eps: float = 1e-5
    rope_base: float = 10000.0
    causal: bool = True
    # zero-padded layouts (exactly equivalent to the unpadded model): a true head size below
    # head_dim (Qwen2.5-VL ViT: 80 in a 128-wide head, laid out [h/2 real | pad | h/2 real | pad]
    # so rotate-half pairs never mix real and pad dims) and a true FFN width below ffn (3420 in
    # 3456: TMA row pitches are 16-byte multiples and the SwiGLU epilogue works on 32-feature blocks)
    head_dim_true: int = 0
    ffn_true: int = 0

    @property
    def hd_true(self) -> int:
        return self.head_dim_true or self.head_dim

    @property
    def ffn_real(self) -> int:
        return self.ffn_true or self.ffn

    @property
    def qkv_dim(self) -> int:
        return (self.heads + 2 * self.kv_heads) * self.head_dim

    def param_shapes(self):
        out = [("embed", (self.vocab, self.d))]
        for i in range(self.layers):
            out += [
                (f"l{i}.ln1", (self.d,)), (f"l{i}.wqkv", (self.qkv_dim, self.d)),
                (f"l{i}.wo", (self.d, self.heads * self.head_dim)), (f"l{i}.ln2", (self.d,)),
                (f"l{i}.wgu", (2 * self.ffn, self.d)), (f"l{i}.wd", (self.d, self.ffn)),
            ]
        out.append(("lnf", (self.d,)))
        if not self.tied:
            out.append(("head", (self.vocab, self.d)))
        return out

    def n_params(self) -> int:
        return sum(math.prod(s) for _, s in self.param_shapes())

    def fwd_flops_per_token(self, seq_len: int, with_head: bool = True) -> float:
        """Model FLOPs of one forward token (GEMMs + causal attention at seq_len)."""
        hd, F = self.hd_true, self.ffn_real  # algorithmic FLOPs of the unpadded model
        lin = self.layers * (self.d * (self.heads + 2 * self.kv_heads) * hd + self.heads * hd * self.d
                             + 3 * self.d * F)
        attn = self.layers * 4 * self.heads * hd * seq_len * (0.5 if self.causal else 1.0)
        head = self.vocab * self.d if with_head else 0
        return 2.0 * (lin + head) + attn


SHAPES = {
    # cfg 2: TinyLlama-1.1B-shaped teacher, 125M-class student (tied embeddings)
    "kd_teacher_1b": Shape(d=2048, layers=22, heads=32, kv_heads=4, ffn=5632, vocab=32000),
    "kd_student_125m": Shape(d=768, layers=12, heads=12, kv_heads=12, ffn=3072, vocab=32000, tied=True),
    # cfg 1: 2-layer GPT backbone (d=768) and ViT-tiny encoder (bidirectional, no vocab)
    "vlm_gpt2l": Shape(d=768, layers=2, heads=12, kv_heads=12, ffn=3072, vocab=32768),
    "vit_tiny": Shape(d=192, layers=12, heads=3, kv_heads=3, ffn=768, vocab=8, causal=False),
    # cfg 5: Llama-3-8B-shaped teacher (head_dim 128, GQA 32/8), Llama-3.2-1B-shaped student (tied)
    "llama3_8b": Shape(d=4096, layers=32, heads=32, kv_heads=8, ffn=14336, vocab=128256, head_dim=128,
                       rope_base=500000.0),
    "llama32_1b": Shape(d=2048, layers=16, heads=32, kv_heads=8, ffn=8192, vocab=128256, tied=True,
                        rope_base=500000.0),
    # tiny shapes for tests
    "test_tiny": Shape(d=128, layers=2, heads=2, kv_heads=1, ffn=256, vocab=512),
    "test_tiny_hd128": Shape(d=256, layers=2, heads=4, kv_heads=2, ffn=512, vocab=512, head_dim=128,
                             rope_base=500000.0),
}


def _align(n: int, a: int = 64) -> int:
    return (n + a - 1) // a * a


class FlatParams:
    """Parameters of one section in contiguous arenas."""

    def __init__(self, shapes, device, trainable: bool, seed: int, std: float = 0.02):
        self.index = {}
        off = 0
        for name, shp in shapes:
            n = math.prod(shp)
            self.index[name] = (off, shp)
            off += _align(n)
        self.numel = _align(off, 256)
        self.trainable = trainable
        g = torch.Generator(device=device).manual_seed(seed)
        master = torch.empty(self.numel, device=device, dtype=torch.float32)
        master.normal_(0.0, std, generator=g)
        for name, (o, shp) in self.index.items():
            if len(shp) == 1:  # norm gains
                master[o: o + shp[0]] = 1.0
        self.w = master.to(torch.bfloat16)
        if trainable:
            self.master = master
            self.grad = torch.zeros_like(master)
            self.m = torch.zeros_like(master)
            self.v = torch.zeros_like(master)
        else:
            del master
            self.master = self.grad = self.m = self.v = None
        self.step = 0
        # K-major (transposed) bf16 copies of the trainable matrices: the dgrad GEMM then reads
        # its B operand K-major, which admits the 256 x 192 tile that fits 768-wide outputs
        self.wt = {}
        if trainable:
            for name, (o, shp) in self.index.items():
                if len(shp) == 2:
                    self.wt[name] = torch.empty(shp[1], shp[0], device=device, dtype=torch.bfloat16)
            self.refresh_transposed()

    def _view(self, buf, name):
        o, shp = self.index[name]
        return buf[o: o + math.prod(shp)].view(*shp)

    def __getitem__(self, name):
        return self._view(self.w, name)

    def g(self, name):
        return self._view(self.grad, name)

    def t(self, name):
        """Transposed bf16 copy [in, out] of a trainable matrix (None when not kept)."""
        return self.wt.get(name)

    def refresh_transposed(self):
        """Re-derive every K-major weight copy from the updated bf16 weights: one launch for all
        (the descriptor table is built once; the arenas are never reallocated)."""
        if not self.wt:
            return
        if getattr(self, "_tdesc", None) is None or self._tdesc_n != len(self.wt):
            self._tdesc, self._ttiles = K.transpose_batch_desc([(self[n], wt) for n, wt in self.wt.items()],
                                                               self.w.device)
            self._tdesc_n = len(self.wt)
        K.transpose_batched(self._tdesc, self._ttiles)

    def zero_grad(self):
        self.grad.zero_()

    def adamw(self, lr: float, wd: float = 0.1, gscale: float = 1.0):
        self.step += 1
        K.adamw(self.master, self.grad, self.m, self.v, self.w, lr, self.step, wd=wd, gscale=gscale)
        self.refresh_transposed()


def rope_table(max_pos: int, head_dim: int, base: float, device, true_dim: int = 0) -> torch.Tensor:
    """(cos, sin) of every (position, frequency) in the position-tiled layout the kernels read:
    [ceil(P/32)][head_dim/2][32 positions][2] fp32 (include/maestro_b200.h).  A warp's 32 rows
    are 32 consecutive positions, so each per-frequency read is one contiguous 256-byte segment.
    ``true_dim`` < head_dim (zero-padded heads): pair i < true_dim/2 gets the true model's
    frequency base^(-2i/true_dim); the pad pairs get frequency 0 (identity rotation of zeros)."""
    half = head_dim // 2
    P = (max_pos + 31) // 32 * 32
    td = true_dim or head_dim
    inv = base ** (-torch.arange(0, head_dim, 2, dtype=torch.float64) / td)
    inv[td // 2:] = 0.0
    ang = torch.arange(P, dtype=torch.float64)[:, None] * inv[None, :]  # [P, half]
    cs = torch.stack([ang.cos(), ang.sin()], -1).to(torch.float32)      # [P, half, 2]
    return cs.view(P // 32, 32, half, 2).transpose(1, 2).contiguous().to(device)


def pad_masks(shape: Shape, device):
    """Boolean masks of the padding of a zero-padded shape: (qkv rows [qkv_dim], wo columns
    [H*dh], gate/up rows [2F], wd columns [F]); True = pad (always zero)."""
    dh, ht = shape.head_dim, shape.hd_true // 2
    j = torch.arange(dh, device=device)
    head_pad = (j % (dh // 2)) >= ht  # [real h/2 | pad | real h/2 | pad]
    qkv = head_pad.repeat(shape.heads + 2 * shape.kv_heads)
    wo = head_pad.repeat(shape.heads)
    f = torch.arange(shape.ffn, device=device)
    fpad = f >= shape.ffn_real
    gu = torch.empty(2 * shape.ffn, dtype=torch.bool, device=device)
    gi = (f // 32) * 64 + f % 32  # gate row of feature f; its up row is gi + 32
    gu[gi] = fpad
    gu[gi + 32] = fpad
    return qkv, wo, gu, fpad


def zero_padding(shape: Shape, p: "FlatParams") -> None:
    """Zero the pad rows / columns of every layer (master, working copy, transposed copies).
    Their gradients are exactly zero (the pad activations are zero and feed nothing), so AdamW
    keeps them at zero and the padded model stays equivalent to the unpadded one."""
    qkv, wo, gu, fpad = pad_masks(shape, p.w.device)
    bufs = [p.w] + ([p.master] if p.master is not None else [])
    for i in range(shape.layers):
        for buf in bufs:
            p._view(buf, f"l{i}.wqkv")[qkv] = 0
            p._view(buf, f"l{i}.wo")[:, wo] = 0
            p._view(buf, f"l{i}.wgu")[gu] = 0
            p._view(buf, f"l{i}.wd")[:, fpad] = 0
    p.refresh_transposed()


@dataclass
class Batch:
    """One packed micro-batch: token ids [T] int32, cu_seqlens [n+1] int32, positions [T]."""

    ids: torch.Tensor
    cu: torch.Tensor
    pos: torch.Tensor
    max_len: int

    @property
    def T(self) -> int:
        return self.pos.shape[0]


class Transformer:
    """Explicit fwd/bwd of a decoder (or, with causal=False, encoder) stack."""

    def __init__(self, shape: Shape, params: FlatParams, device, max_pos: int = 8192):
        self.s = shape
        self.p = params
        self.device = device
        self.cs = rope_table(max_pos, shape.head_dim, shape.rope_base, device, shape.hd_true)
        self.scale = 1.0 / math.sqrt(shape.hd_true)
        if shape.hd_true != shape.head_dim or shape.ffn_real != shape.ffn:
            zero_padding(shape, params)

    # -------------------------------------------------------------------- forward
    def forward(self, b: Batch, x0: torch.Tensor | None = None, save: bool = True, yf_out: torch.Tensor | None = None):
        """Returns (yf [T, d] final-normed hidden, ctx for backward).  x0 overrides the embedding;
        ``yf_out`` receives the final hidden state (e.g. rows of a handoff buffer)."""
        s, p, T = self.s, self.p, b.T
        dev, bf = self.device, torch.bfloat16
        if x0 is None:
            x0 = torch.empty(T, s.d, device=dev, dtype=bf)
            K.embed(p["embed"], b.ids, x0)
        ctx = {"b": b, "layers": [], "x0": x0, "plan": A.plan(b.cu, T)}  # tile lists, once per micro-batch
        x = x0  # residual stream entering the block (h1); the residual adds run in GEMM epilogues
        H, Hk, dh = s.heads, s.kv_heads, s.head_dim
        for i in range(s.layers):
            h1 = x
            y1 = torch.empty(T, s.d, device=dev, dtype=bf)
            r1 = torch.empty(T, device=dev, dtype=torch.float32)
            K.add_rmsnorm(h1, None, h1, y1, p[f"l{i}.ln1"], r1, s.eps)
            # QKV projection with RoPE fused into the GEMM epilogue (one head per 64-col chunk)
            qkv = D.linear_fwd_rope(y1, p[f"l{i}.wqkv"], b.pos, self.cs, (H + Hk) * dh, head_dim=dh)
            q = qkv[:, : H * dh].view(T, H, dh)
            k = qkv[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
            v = qkv[:, (H + Hk) * dh:].view(T, Hk, dh)
            o = torch.empty(T, H, dh, device=dev, dtype=bf)
            lse = A.attn_fwd(q, k, v, b.cu, b.max_len, s.causal, o, self.scale, plan=ctx["plan"])
            # h2 = h1 + o Wo^T (residual add in the epilogue)
            h2 = D.linear_fwd_residual(o.view(T, H * dh), p[f"l{i}.wo"], h1)
            y2 = torch.empty(T, s.d, device=dev, dtype=bf)
            r2 = torch.empty(T, device=dev, dtype=torch.float32)
            K.add_rmsnorm(h2, None, h2, y2, p[f"l{i}.ln2"], r2, s.eps)
            # gate/up projection with SwiGLU fused into the epilogue (gate/up rows interleaved
            # in 32-row blocks in wgu)
            sw = torch.empty(T, s.ffn, device=dev, dtype=bf)
            gu = D.linear_fwd_swiglu(y2, p[f"l{i}.wgu"], sw, store_gu=save)  # gu only kept for backward
            if save:
                ctx["layers"].append((h1, r1, y1, qkv, o, lse, h2, r2, y2, gu, sw))
            # next block's residual stream: h2 + sw Wd^T
            x = D.linear_fwd_residual(sw, p[f"l{i}.wd"], h2)
        hf = x
        yf = torch.empty(T, s.d, device=dev, dtype=bf) if yf_out is None else yf_out
        rf = torch.empty(T, device=dev, dtype=torch.float32)
        K.add_rmsnorm(hf, None, hf, yf, p["lnf"], rf, s.eps)
        ctx["final"] = (hf, rf, yf)
        return yf, ctx

    def head_weight(self):
        return self.p["embed"] if self.s.tied else self.p["head"]

    def logits(self, yf: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        return D.linear_fwd(yf, self.head_weight(), out)

    # -------------------------------------------------------------------- backward
    def backward(self, ctx, dlogits: torch.Tensor | None = None, dyf: torch.Tensor | None = None,
                 need_dx0: bool = False, dyf_hook=None, layer_hook=None):
        """Accumulates parameter grads (fp32) from dlogits (or dyf); returns dx0 if asked.
        ``dyf_hook(dyf)`` may add further gradient into the final hidden state's gradient (e.g. a
        downstream section's) before the stack's backward; ``layer_hook(i)`` runs (on the current
        stream) once layer i's parameter gradients of this call have been enqueued -- the per-layer
        buckets of an overlapped gradient all-reduce (gradsync.GradSync)."""
        s, p, b = self.s, self.p, ctx["b"]
        T, dev, bf = b.T, self.device, torch.bfloat16
        H, Hk, dh = s.heads, s.kv_heads, s.head_dim
        hf, rf, yf = ctx["final"]
        if dlogits is not None:
            hw = "embed" if s.tied else "head"
            dyf = D.linear_dgrad(dlogits, p[hw], wt=p.t(hw))
            D.linear_wgrad(dlogits, yf, p.g(hw))
        if dyf_hook is not None:
            dyf_hook(dyf)
        dh_ = torch.empty(T, s.d, device=dev, dtype=bf)
        K.rmsnorm_bwd(dyf, hf, p["lnf"], rf, None, dh_, p.g("lnf"))
        if layer_hook is not None:
            layer_hook(-1)  # the output head (untied) and the final norm are final from here
        for i in reversed(range(s.layers)):
            h1, r1, y1, qkv, o, lse, h2, r2, y2, gu, sw = ctx["layers"][i]
            # MLP
            dsw = D.linear_dgrad(dh_, p[f"l{i}.wd"], wt=p.t(f"l{i}.wd"))
            D.linear_wgrad(dh_, sw, p.g(f"l{i}.wd"))
            dgu = torch.empty_like(gu)
            K.swiglu_bwd(dsw, gu, dgu)
            D.linear_wgrad(dgu, y2, p.g(f"l{i}.wgu"))
            dy2 = D.linear_dgrad(dgu, p[f"l{i}.wgu"], wt=p.t(f"l{i}.wgu"))
            dh2 = torch.empty(T, s.d, device=dev, dtype=bf)
            K.rmsnorm_bwd(dy2, h2, p[f"l{i}.ln2"], r2, dh_, dh2, p.g(f"l{i}.ln2"))
            # attention
            do = D.linear_dgrad(dh2, p[f"l{i}.wo"], wt=p.t(f"l{i}.wo"))
            D.linear_wgrad(dh2, o.view(T, H * dh), p.g(f"l{i}.wo"))
            dqkv = torch.empty_like(qkv)
            q = qkv[:, : H * dh].view(T, H, dh)
            k = qkv[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
            v = qkv[:, (H + Hk) * dh:].view(T, Hk, dh)
            dq = dqkv[:, : H * dh].view(T, H, dh)
            dk = dqkv[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
            dv = dqkv[:, (H + Hk) * dh:].view(T, Hk, dh)
            # inverse RoPE fused into the attention backward's dQ / dK stores
            A.attn_bwd(do.view(T, H, dh), q, k, v, o, lse, b.cu, b.max_len, s.causal, dq, dk, dv, self.scale,
                       rope=(b.pos, self.cs), plan=ctx["plan"])
            D.linear_wgrad(dqkv, y1, p.g(f"l{i}.wqkv"))
            dy1 = D.linear_dgrad(dqkv, p[f"l{i}.wqkv"], wt=p.t(f"l{i}.wqkv"))
            dh1 = torch.empty(T, s.d, device=dev, dtype=bf)
            K.rmsnorm_bwd(dy1, h1, p[f"l{i}.ln1"], r1, dh2, dh1, p.g(f"l{i}.ln1"))
            dh_ = dh1
            if layer_hook is not None:
                layer_hook(i)
        if need_dx0:
            return dh_
        K.embed_bwd(dh_, b.ids, p.g("embed"))
        return None
