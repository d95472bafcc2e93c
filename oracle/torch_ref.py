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


def forward(shape, P, ids, cu, x0=None):
    """fp32 forward of the stack -> final normed hidden [T, d]."""
    T = ids.shape[0]
    x = P["embed"][ids.long()] if x0 is None else x0
    cu_l = cu.tolist()
    pos = torch.cat([torch.arange(b - a, device=ids.device) for a, b in zip(cu_l[:-1], cu_l[1:])])
    H, Hk, dh = shape.heads, shape.kv_heads, shape.head_dim
    scale = 1.0 / math.sqrt(dh)
    for i in range(shape.layers):
        y = rms_norm(x, P[f"l{i}.ln1"], shape.eps)
        qkv = y @ P[f"l{i}.wqkv"].t()
        q = qkv[:, : H * dh].view(T, H, dh)
        k = qkv[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
        v = qkv[:, (H + Hk) * dh:].view(T, Hk, dh)
        q, k = rope(q, pos, shape.rope_base), rope(k, pos, shape.rope_base)
        o = varlen_attention(q, k, v, cu, shape.causal, scale)
        x = x + o.reshape(T, H * dh) @ P[f"l{i}.wo"].t()
        y = rms_norm(x, P[f"l{i}.ln2"], shape.eps)
        gu = y @ P[f"l{i}.wgu"].t()
        g, u = gu[:, gate_index(shape.ffn, gu.device)], gu[:, gate_index(shape.ffn, gu.device) + 32]
        x = x + (F.silu(g) * u) @ P[f"l{i}.wd"].t()
    return rms_norm(x, P["lnf"], shape.eps)


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


def kd_step_reference(tshape, sshape, t_flat, s_flat, t_head, ids, cu, global_tokens):
    """One KD micro-batch in fp32 autograd: returns (sum of token KL, student grads flat)."""
    Pt = param_views(tshape, t_flat)
    s_flat = s_flat.detach().clone().requires_grad_(True)
    Ps = param_views(sshape, s_flat)
    with torch.no_grad():
        t_logits = forward(tshape, Pt, ids, cu) @ t_head.t()
    s_logits = forward(sshape, Ps, ids, cu) @ head_weight(sshape, Ps).t()
    tok = kd_loss(t_logits, s_logits)
    (tok.sum() / global_tokens).backward()
    return tok.detach(), s_flat.grad


def adamw_reference(p, g, m, v, lr, step, b1=0.9, b2=0.95, eps=1e-8, wd=0.1):
    m.mul_(b1).add_(g, alpha=1 - b1)
    v.mul_(b2).addcmul_(g, g, value=1 - b2)
    upd = (m / (1 - b1 ** step)) / ((v / (1 - b2 ** step)).sqrt() + eps)
    p.sub_(lr * (upd + wd * p))
    return p


def vlm_step_reference(llm_shape, vit_shape, llm_flat, vit_flat, hb, merge_idx, patch_dim=768):
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
        x0 = px @ Pv["patch_w"].t()
        cu = torch.arange(0, n_img * 196 + 1, 196, dtype=torch.int32, device=dev)
        yf = forward(vit_shape, Pv, torch.zeros(n_img * 196, dtype=torch.int32, device=dev), cu, x0=x0)
        src = (torch.from_numpy(merge_idx).to(dev)[None, :].long() + 196 * torch.arange(n_img, device=dev)[:, None]).reshape(-1)
        merged = yf[src].view(n_img * 49, 4 * vit_shape.d)
        emb = merged @ Pv["proj_w"].t()
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
        y = forward(llm_shape, Pl, ids, cu, x0=x)
        logits = y @ head_weight(llm_shape, Pl).t()
        valid = lab >= 0
        if valid.any():
            loss_sum = loss_sum + F.cross_entropy(logits[valid], lab[valid], reduction="sum")
            nlab += int(valid.sum())
    loss = loss_sum / max(nlab, 1)
    loss.backward()
    return loss.item(), lf.grad, vf.grad
