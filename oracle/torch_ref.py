"""ORACLE -- test infrastructure only.

Plain PyTorch fp32 restatement of the section compute (Llama-style block, RoPE, SwiGLU, varlen
causal attention, full-vocab KL distillation, AdamW).  The reference has no GPU code and no
model code at all: these semantics come from the paper prose (KL distillation PAPER.md:93,
242, 270-271; forward-only teacher PAPER.md:72; colocated teacher head workload.py:471-514;
4:1 merged visual tokens concatenated with text PAPER.md:56,250), so parity for this part is
"unpinned by the reference" and is checked against this fp32 restatement with stated
tolerances.  Used by tests (numerics) and by bench.py's cpu_baseline / --impl reference leg
(timed on CPU with all host threads).  Never imported by the product package.
"""

from __future__ import annotations

import math

import numpy as np

import torch
import torch.nn.functional as F


def rms_norm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def rope(x, pos, base):
    """x [T, H, dh]; rotate-half convention on pairs (i, i + dh/2)."""
    dh = x.shape[-1]
    inv = base ** (-torch.arange(0, dh, 2, dtype=torch.float64, device=x.device) / dh)
    ang = pos.double()[:, None] * inv[None, :]
    c, s = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]
    a, b = x[..., : dh // 2], x[..., dh // 2:]
    return torch.cat([a * c - b * s, b * c + a * s], -1)


def varlen_attention(q, k, v, cu, causal, scale):
    """q [T,H,dh], k/v [T,Hk,dh]; per-sequence softmax attention (GQA by head repetition)."""
    T, H, dh = q.shape
    Hk = k.shape[1]
    rep = H // Hk
    out = torch.empty_like(q)
    cu = cu.tolist()
    for a, b in zip(cu[:-1], cu[1:]):
        qs = q[a:b].transpose(0, 1)
        ks = k[a:b].repeat_interleave(rep, 1).transpose(0, 1)
        vs = v[a:b].repeat_interleave(rep, 1).transpose(0, 1)
        s = (qs @ ks.transpose(1, 2)) * scale
        if causal:
            n = b - a
            mask = torch.ones(n, n, dtype=torch.bool, device=q.device).triu(1)
            s = s.masked_fill(mask, float("-inf"))
        out[a:b] = (s.softmax(-1) @ vs).transpose(0, 1)
    return out


def param_views(shape, flat):
    """Split a flat fp32 parameter vector using the product's arena layout (same offsets)."""
    out = {}
    off = 0
    for name, shp in shape.param_shapes():
        n = math.prod(shp)
        out[name] = flat[off: off + n].view(*shp)
        off += (n + 63) // 64 * 64
    return out


def rb(t, on=True):
    """Straight-through bf16 rounding: the forward value is rounded to bf16 (where the kernels
    store an activation in bf16), the gradient passes through in fp32."""
    return t + (t.bfloat16().float() - t).detach() if on else t


def forward(shape, P, ids, cu, x0=None, bf16=False):
    """fp32 forward of the stack -> final normed hidden [T, d].  ``bf16``: round activations at
    the points where the kernels store them in bf16 (norm outputs, the RoPE'd QKV, attention
    output, the residual stream after each fused residual-add epilogue, the SwiGLU output and the
    final hidden), so only accumulation order separates the two -- the rounding-aware oracle."""
    T = ids.shape[0]
    x = P["embed"][ids.long()] if x0 is None else x0
    cu_l = cu.tolist()
    pos = torch.cat([torch.arange(b - a, device=ids.device) for a, b in zip(cu_l[:-1], cu_l[1:])])
    H, Hk, dh = shape.heads, shape.kv_heads, shape.head_dim
    scale = 1.0 / math.sqrt(dh)
    for i in range(shape.layers):
        y = rb(rms_norm(x, P[f"l{i}.ln1"], shape.eps), bf16)
        qkv = y @ P[f"l{i}.wqkv"].t()
        q = qkv[:, : H * dh].view(T, H, dh)
        k = qkv[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
        v = rb(qkv[:, (H + Hk) * dh:].view(T, Hk, dh), bf16)
        q, k = rb(rope(q, pos, shape.rope_base), bf16), rb(rope(k, pos, shape.rope_base), bf16)
        o = rb(varlen_attention(q, k, v, cu, shape.causal, scale), bf16)
        x = rb(x + o.reshape(T, H * dh) @ P[f"l{i}.wo"].t(), bf16)
        y = rb(rms_norm(x, P[f"l{i}.ln2"], shape.eps), bf16)
        gu = y @ P[f"l{i}.wgu"].t()
        g, u = gu[:, gate_index(shape.ffn, gu.device)], gu[:, gate_index(shape.ffn, gu.device) + 32]
        x = rb(x + rb(F.silu(g) * u, bf16) @ P[f"l{i}.wd"].t(), bf16)
    return rb(rms_norm(x, P["lnf"], shape.eps), bf16)


def gate_index(F, device):
    """Columns of the gate features in the interleaved [g(32) | u(32)] gate/up layout."""
    f = torch.arange(F, device=device)
    return (f // 32) * 64 + f % 32


def head_weight(shape, P):
    return P["embed"] if shape.tied else P["head"]


def kd_loss(t_logits, s_logits, tau=1.0):
    """Per-token KL(softmax(t/tau) || softmax(s/tau))."""
    lt = F.log_softmax(t_logits.float() / tau, -1)
    ls = F.log_softmax(s_logits.float() / tau, -1)
    return (lt.exp() * (lt - ls)).sum(-1)


def kd_step_reference(tshape, sshape, t_flat, s_flat, t_head, ids, cu, global_tokens, bf16=False):
    """One KD micro-batch in fp32 autograd: returns (sum of token KL, student grads flat).
    ``bf16``: the rounding-aware forward (see forward); logits rounded like the GEMM outputs."""
    Pt = param_views(tshape, t_flat)
    s_flat = s_flat.detach().clone().requires_grad_(True)
    Ps = param_views(sshape, s_flat)
    with torch.no_grad():
        t_logits = rb(forward(tshape, Pt, ids, cu, bf16=bf16) @ t_head.t(), bf16)
    s_logits = rb(forward(sshape, Ps, ids, cu, bf16=bf16) @ head_weight(sshape, Ps).t(), bf16)
    tok = kd_loss(t_logits, s_logits)
    (tok.sum() / global_tokens).backward()
    return tok.detach(), s_flat.grad


def adamw_reference(p, g, m, v, lr, step, b1=0.9, b2=0.95, eps=1e-8, wd=0.1):
    m.mul_(b1).add_(g, alpha=1 - b1)
    v.mul_(b2).addcmul_(g, g, value=1 - b2)
    upd = (m / (1 - b1 ** step)) / ((v / (1 - b2 ** step)).sqrt() + eps)
    p.sub_(lr * (upd + wd * p))
    return p


def vlm_step_reference(llm_shape, vit_shape, llm_flat, vit_flat, hb, merge_idx, patch_dim=768, bf16=False):
    """fp32 autograd restatement of one VLM step (ViT -> 2x2 merge -> projector -> scatter into the
    LLM sequence at the placeholder offset -> LLM -> next-token CE).  Returns (loss, llm grad, vit grad)."""
    dev = llm_flat.device
    lf = llm_flat.detach().clone().requires_grad_(True)
    vf = vit_flat.detach().clone().requires_grad_(True)
    Pl = param_views(llm_shape, lf)
    extra = [("patch_w", (vit_shape.d, patch_dim)), ("proj_w", (llm_shape.d, 4 * vit_shape.d))]

    class _S:  # vit shape + extra params
        pass

    Pv = {}
    off = 0
    for name, shp in vit_shape.param_shapes() + extra:
        n = math.prod(shp)
        Pv[name] = vf[off: off + n].view(*shp)
        off += (n + 63) // 64 * 64
    n_img = hb["pixels"].shape[0]
    emb = None
    if n_img:
        px = torch.from_numpy(hb["pixels"]).to(dev).to(torch.bfloat16).float().view(-1, patch_dim)
        x0 = rb(px @ Pv["patch_w"].t(), bf16)
        cu = torch.arange(0, n_img * 196 + 1, 196, dtype=torch.int32, device=dev)
        yf = forward(vit_shape, Pv, torch.zeros(n_img * 196, dtype=torch.int32, device=dev), cu, x0=x0, bf16=bf16)
        src = (torch.from_numpy(merge_idx).to(dev)[None, :].long() + 196 * torch.arange(n_img, device=dev)[:, None]).reshape(-1)
        merged = yf[src].view(n_img * 49, 4 * vit_shape.d)
        emb = rb(merged @ Pv["proj_w"].t(), bf16)
    total, nlab = 0.0, 0
    loss_sum = torch.zeros((), device=dev)
    for i in range(hb["ids"].shape[0]):
        L = int(hb["lens"][i])
        ids = torch.from_numpy(hb["ids"][i, :L]).to(dev)
        lab = torch.from_numpy(hb["labels"][i, :L]).to(dev).long()
        x = Pl["embed"][ids.clamp_min(0).long()] * (ids >= 0).float()[:, None]
        if hb["has_img"][i]:
            o = int(hb["img_offset"][i])
            k = int(hb["img_ordinal"][i])
            x = torch.cat([x[:o], emb[49 * k: 49 * k + 49], x[o + 49:]], 0)
        cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
        y = forward(llm_shape, Pl, ids, cu, x0=x, bf16=bf16)
        logits = rb(y @ head_weight(llm_shape, Pl).t(), bf16)
        valid = lab >= 0
        if valid.any():
            loss_sum = loss_sum + F.cross_entropy(logits[valid], lab[valid], reduction="sum")
            nlab += int(valid.sum())
    loss = loss_sum / max(nlab, 1)
    loss.backward()
    return loss.item(), lf.grad, vf.grad


# ------------------------------------------------------------------------------------------------
# Generic section graph (graph_exec.SectionGraphExecutor): encoders -> backbone -> decoders
def unpad_heads(shape, P):
    """A zero-padded-head shape (head_dim_true < head_dim, real dims laid out [h/2 | pad | h/2 |
    pad]) -> the true model's (shape, params): the standard rotate-half RoPE over h dims with
    base^(-2i/h) and scale 1/sqrt(h) -- the model the padded layout must equal."""
    import dataclasses

    ht, dh = shape.hd_true, shape.head_dim
    if ht == dh:
        return shape, P
    keep = torch.cat([torch.arange(ht // 2), dh // 2 + torch.arange(ht // 2)])
    nq = shape.heads + 2 * shape.kv_heads
    rows = (torch.arange(nq)[:, None] * dh + keep[None, :]).reshape(-1)
    cols = (torch.arange(shape.heads)[:, None] * dh + keep[None, :]).reshape(-1)
    Q = dict(P)
    for i in range(shape.layers):
        Q[f"l{i}.wqkv"] = P[f"l{i}.wqkv"][rows.to(P[f"l{i}.wqkv"].device)]
        Q[f"l{i}.wo"] = P[f"l{i}.wo"][:, cols.to(P[f"l{i}.wo"].device)]
    return dataclasses.replace(shape, head_dim=ht, head_dim_true=0), Q


def views(shape, flat, extra=()):
    """Arena views (same offsets as FlatParams) of shape.param_shapes() + extra."""
    out, off = {}, 0
    for name, shp in list(shape.param_shapes()) + list(extra):
        n = math.prod(shp)
        out[name] = flat[off: off + n].view(*shp)
        off += (n + 63) // 64 * 64
    return out


def graph_step_reference(crit, ups, downs, gb, bf16=False):
    """fp32 autograd restatement of one generic-executor step over the WHOLE batch (sample order
    does not matter: training equivalence).

    crit  = (shape, flat)                      backbone, next-token CE over gb.labels
    ups   = {name: (shape, flat, in_dim, merge)}  encoder: in_w -> stack -> 4:1 merge -> proj_w
    downs = {name: (shape, flat, in_d)}        decoder: in_w -> causal stack -> head -> CE
    Returns (loss, {name: flat grad}).  Loss = mean CE of the backbone + mean CE of each decoder."""
    dev = crit[1].device
    leaves = {}
    cs, cflat = crit
    lf = cflat.detach().clone().requires_grad_(True)
    leaves["crit"] = lf
    Pc = param_views(cs, lf)
    enc_rows = {}
    for name, (sh, flat, in_dim, merge) in ups.items():
        vf = flat.detach().clone().requires_grad_(True)
        leaves[name] = vf
        P = views(sh, vf, [("in_w", (sh.d, in_dim)), ("proj_w", (cs.d, merge * sh.d))])
        ui = gb.up[name]
        act = [i for i in range(gb.B) if ui.in_len[i] > 0]
        rows = {}
        if act:
            feats = torch.from_numpy(ui.feats).to(dev).to(torch.bfloat16).float()
            fo = np.concatenate([[0], np.cumsum(ui.in_len)]).astype(np.int64)
            sh_t, Pt = unpad_heads(sh, P)
            for i in act:
                x = rb(feats[fo[i]: fo[i + 1]] @ P["in_w"].t(), bf16)
                cu = torch.tensor([0, int(ui.in_len[i])], dtype=torch.int32, device=dev)
                y = forward(sh_t, Pt, torch.zeros(int(ui.in_len[i]), dtype=torch.int32, device=dev), cu, x0=x,
                            bf16=bf16)
                rows[i] = rb(y.reshape(-1, merge * sh.d) @ P["proj_w"].t(), bf16)
        enc_rows[name] = rows
    dec = {}
    for name, (sh, flat, in_d) in downs.items():
        vf = flat.detach().clone().requires_grad_(True)
        leaves[name] = vf
        dec[name] = (sh, views(sh, vf, [("in_w", (sh.d, in_d))]))
    cs_t, Pc_t = unpad_heads(cs, Pc)
    n_lab = max(int((gb.labels >= 0).sum()), 1)
    loss = torch.zeros((), device=dev)
    dec_sum = {n: torch.zeros((), device=dev) for n in downs}
    for i in range(gb.B):
        L = int(gb.lens[i])
        ids = torch.from_numpy(gb.ids[i, :L]).to(dev)
        lab = torch.from_numpy(gb.labels[i, :L]).to(dev).long()
        x = Pc["embed"][ids.clamp_min(0).long()] * (ids >= 0).float()[:, None]
        for name in ups:
            if i in enc_rows[name]:
                o = int(gb.up[name].dst_off[i])
                r = enc_rows[name][i]
                x = torch.cat([x[:o], r, x[o + r.shape[0]:]], 0)
        cu = torch.tensor([0, L], dtype=torch.int32, device=dev)
        y = forward(cs_t, Pc_t, ids, cu, x0=x, bf16=bf16)
        logits = rb(y @ head_weight(cs, Pc).t(), bf16)
        valid = lab >= 0
        if valid.any():
            loss = loss + F.cross_entropy(logits[valid], lab[valid], reduction="sum") / n_lab
        for name, (sh, P) in dec.items():
            di = gb.down[name]
            nr = int(di.rows[i])
            if nr == 0:
                continue
            so = int(di.src_off[i])
            t_off = int(np.sum(di.rows[:i]))
            tg = torch.from_numpy(di.targets[t_off: t_off + nr]).to(dev).long()
            xin = rb(y[so: so + nr] @ P["in_w"].t(), bf16)
            cu_d = torch.tensor([0, nr], dtype=torch.int32, device=dev)
            yd = forward(sh, P, torch.zeros(nr, dtype=torch.int32, device=dev), cu_d, x0=xin, bf16=bf16)
            dec_sum[name] = dec_sum[name] + F.cross_entropy(rb(yd @ head_weight(sh, P).t(), bf16), tg,
                                                            reduction="sum")
    for name in downs:
        loss = loss + dec_sum[name] / max(int(gb.down[name].rows.sum()), 1)
    loss.backward()
    return loss.item(), {k: v.grad for k, v in leaves.items()}
