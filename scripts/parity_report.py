"""Parity report: error of the CUDA path against the fp32 oracle and the bf16-rounding-aware
oracle (oracle/torch_ref.forward(bf16=True)), as max-normalised max error and relative L2 norm,
for the transformer (hd 64/128), the KD step and the generic executor (cfg 3 / cfg 4 structure).
Writes gpurun_out/parity_report.json."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from oracle import torch_ref as R  # noqa: E402


def errs(a, b):
    a, b = a.float(), b.float()
    return {"maxnorm": ((a - b).abs().max() / b.abs().max().clamp_min(1e-12)).item(),
            "relnorm": ((a - b).norm() / b.norm().clamp_min(1e-12)).item()}


def transformer(shape_name, causal):
    import dataclasses

    from paper_2605_10501_b200 import kernels as K
    from paper_2605_10501_b200.transformer import SHAPES, Batch, FlatParams, Transformer

    shape = dataclasses.replace(SHAPES[shape_name], causal=causal)
    p = FlatParams(shape.param_shapes(), torch.device("cuda"), trainable=True, seed=3)
    model = Transformer(shape, p, torch.device("cuda"), max_pos=1024)
    lens = [100, 37, 256, 1]
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
    T = sum(lens)
    torch.manual_seed(0)
    ids = torch.randint(0, shape.vocab, (T,), device="cuda", dtype=torch.int32)
    pos = torch.empty(T, dtype=torch.int32, device="cuda")
    K.positions(cu, len(lens), pos)
    yf, ctx = model.forward(Batch(ids, cu, pos, max(lens)))
    logits = model.logits(yf)
    dl = (torch.randn(T, shape.vocab, device="cuda") * 0.01).bfloat16()
    p.zero_grad()
    model.backward(ctx, dlogits=dl)
    out = {}
    for mode in (False, True):
        flat = p.w.float().clone().requires_grad_(True)
        P = R.param_views(shape, flat)
        yr = R.forward(shape, P, ids, cu, bf16=mode)
        lr_ = R.rb(yr @ R.head_weight(shape, P).t(), mode)
        lr_.backward(dl.float())
        g = R.param_views(shape, flat.grad)
        gp = {n: p.g(n) for n in ("embed", "lnf", "l1.wd", "l1.wgu", "l0.wqkv", "l0.wo", "l0.ln1")}
        out["bf16_oracle" if mode else "fp32_oracle"] = {
            "yf": errs(yf, yr), "logits": errs(logits, lr_),
            **{f"grad:{n}": errs(v, g[n]) for n, v in gp.items()},
            "grad:all": errs(p.grad, flat.grad)}
    return out


def kd_step():
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ex = KDExecutor(n_gpus=1, batch_per_rank=4, seq=128, mbs=2, teacher="test_tiny", student="test_tiny", lr=0.0)
    ids = torch.from_numpy(synthetic_ids(4, 128, 512, seed=5)).cuda()
    t_flat, s_flat = ex.teacher.p.w.float(), ex.student.p.w.float()
    st = ex.step(ids)
    cu = torch.arange(0, 4 * 128 + 1, 128, dtype=torch.int32, device="cuda")
    out = {}
    for mode in (False, True):
        tok, grad = R.kd_step_reference(ex.tshape, ex.sshape, t_flat, s_flat, ex.t_head.float(), ids.reshape(-1), cu,
                                        global_tokens=4 * 128, bf16=mode)
        ref_loss = tok.sum().item() / (4 * 128)
        out["bf16_oracle" if mode else "fp32_oracle"] = {"loss_rel": abs(st.loss - ref_loss) / abs(ref_loss),
                                                         "grad:all": errs(ex.student.p.grad, grad)}
    return out


def vlm_step():
    from paper_2605_10501_b200 import vlm

    ex = vlm.VLMExecutor(batch=12, mbs_llm=4, mbs_vit=3, lr=0.0)
    hb = vlm.vlm_host_batch(12, seed=3)
    lf, vf = ex.llm.p.w.float().clone(), ex.vit.p.w.float().clone()
    st = ex.step(hb)
    out = {}
    for mode in (False, True):
        loss, gl, gv = R.vlm_step_reference(ex.llm_shape, ex.vit_shape, lf, vf, hb, vlm.merge_index(), bf16=mode)
        out["bf16_oracle" if mode else "fp32_oracle"] = {"loss_rel": abs(st.loss - loss) / abs(loss),
                                                         "grad:llm": errs(ex.llm.p.grad, gl),
                                                         "grad:vit": errs(ex.vit.p.grad[: gv.numel()], gv)}
    return out


def graph(kind):
    import test_graph_exec as T

    from paper_2605_10501_b200 import graph_workloads as W
    from paper_2605_10501_b200.graph_exec import BackboneModule, DecoderModule, EncoderModule

    if kind == "vlm7b":
        ex = W.vlm7b_executor(tiny=True, mbs_llm=3, mbs_vit=2, lr=0.0, max_pos=2048)
        gb = W.vlm7b_batch(10, seed=3, vocab=W.TINY_LLM.vocab, patch_dim=128, lo=16, hi=160, text_lo=20, text_hi=90)
    else:
        ex = W.omni_executor(tiny=True, mbs_llm=2, mbs_enc=2, lr=0.0, max_pos=2048)
        gb = W.omni_batch(12, seed=5, vocab=W.TINY_LLM.vocab, patch_dim=128, n_codes=W.TINY_DEC.vocab,
                          img_patches=64, frames=40, dec_rows=12, text_lo=16, text_hi=60, mix="4way")
    T._snapshot(ex)
    st = ex.step(gb)
    crit, ups, downs = None, {}, {}
    for name, m in ex.mod.items():
        if isinstance(m, BackboneModule):
            crit = (m.s, ex._w0[name])
        elif isinstance(m, EncoderModule):
            ups[name] = (m.s, ex._w0[name], m.in_dim, m.merge)
        elif isinstance(m, DecoderModule):
            downs[name] = (m.s, ex._w0[name], m.in_d)
    out = {}
    for mode in (False, True):
        loss, grads = R.graph_step_reference(crit, ups, downs, gb, bf16=mode)
        rec = {"loss_rel": abs(st.loss - loss) / abs(loss)}
        for name, m in ex.mod.items():
            g = grads["crit" if isinstance(m, BackboneModule) else name]
            rec[f"grad:{name}"] = errs(m.p.grad[: g.numel()], g)
        out["bf16_oracle" if mode else "fp32_oracle"] = rec
    return out


def main():
    rep = {}
    for name, fn in [("transformer_hd64_causal", lambda: transformer("test_tiny", True)),
                     ("transformer_hd64_bidir", lambda: transformer("test_tiny", False)),
                     ("transformer_hd128_causal", lambda: transformer("test_tiny_hd128", True)),
                     ("kd_step", kd_step), ("vlm_step", vlm_step), ("graph_vlm7b", lambda: graph("vlm7b")),
                     ("graph_omni4way", lambda: graph("omni"))]:
        try:
            rep[name] = fn()
        except Exception as exc:  # noqa: BLE001
            rep[name] = {"error": repr(exc)}
        print(name, json.dumps(rep[name]), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/parity_report.json").write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
