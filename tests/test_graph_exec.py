"""GPU: the generic section-graph executor (graph_exec) on cfg 3 / cfg 4 / KD structures.

Tiny shapes with the configs' structure: zero-padded 80-in-128 ViT heads and a padded SwiGLU,
GQA backbone, image + audio encoders, a downstream audio decoder.  Every step is checked against
the fp32 autograd restatement of the whole graph in its bf16-rounding-aware mode
(oracle/torch_ref.graph_step_reference(bf16=True); padded heads are compared with the TRUE
unpadded model).  Tolerance: loss within 1e-3 relative; every section's gradient within 1.2e-2
relative L2 and 2e-2 of its max magnitude (measured 7.3e-3 .. 8.8e-3 relative L2,
profiles/r02_parity_report.json).
"""

import numpy as np
import pytest
import torch

from oracle import torch_ref as R

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


def relnorm(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def _check(ex, gb, st, tol=2e-2):
    from paper_2605_10501_b200.graph_exec import BackboneModule, DecoderModule, EncoderModule

    crit = None
    ups, downs = {}, {}
    for name, m in ex.mod.items():
        if isinstance(m, BackboneModule):
            crit = (m.s, ex._w0[name])
        elif isinstance(m, EncoderModule):
            ups[name] = (m.s, ex._w0[name], m.in_dim, m.merge)
        elif isinstance(m, DecoderModule):
            downs[name] = (m.s, ex._w0[name], m.in_d)
    loss, grads = R.graph_step_reference(crit, ups, downs, gb, bf16=True)
    assert abs(st.loss - loss) / abs(loss) < 1e-3, (st.loss, loss)  # measured <= 8e-6
    for name, m in ex.mod.items():
        if not m.trainable:
            continue
        g = grads["crit" if isinstance(m, BackboneModule) else name]
        got = m.p.grad[: g.numel()]
        # measured relative L2 7.3e-3 .. 8.8e-3 (4 sections, 2 layers each, bf16 end to end)
        assert rel(got, g) < tol and relnorm(got, g) < 1.2e-2, (name, rel(got, g), relnorm(got, g))


def _snapshot(ex):
    ex._w0 = {n: m.p.w.float().clone() for n, m in ex.mod.items()}


@pytest.mark.parametrize("policy", ["interleaved", "all-fwd-then-bwd"])
def test_vlm7b_structure_matches_reference(policy):
    from paper_2605_10501_b200 import graph_workloads as W

    ex = W.vlm7b_executor(tiny=True, mbs_llm=3, mbs_vit=2, lr=0.0, policy=policy, max_pos=2048)
    gb = W.vlm7b_batch(10, seed=3, vocab=W.TINY_LLM.vocab, patch_dim=128, lo=16, hi=160, text_lo=20, text_hi=90)
    _snapshot(ex)
    st = ex.step(gb)
    _check(ex, gb, st)
    assert 0.0 <= st.stall_frac <= 1.0


def test_padded_vit_heads_stay_zero_and_exact():
    """80-in-128 heads / 200-in-256 SwiGLU: after a few AdamW steps the pad parameters are still
    exactly zero (their gradients are exactly zero)."""
    from paper_2605_10501_b200 import graph_workloads as W
    from paper_2605_10501_b200.transformer import pad_masks

    ex = W.vlm7b_executor(tiny=True, mbs_llm=4, mbs_vit=4, lr=1e-3, max_pos=2048)
    gb = W.vlm7b_batch(8, seed=4, vocab=W.TINY_LLM.vocab, patch_dim=128, lo=16, hi=96, text_lo=20, text_hi=60)
    for _ in range(3):
        ex.step(gb)
    vit = ex.mod["vit"]
    qkv, wo, gu, fpad = pad_masks(vit.s, "cuda")
    for i in range(vit.s.layers):
        assert torch.all(vit.p[f"l{i}.wqkv"][qkv] == 0) and torch.all(vit.p[f"l{i}.wo"][:, wo] == 0)
        assert torch.all(vit.p[f"l{i}.wgu"][gu] == 0) and torch.all(vit.p[f"l{i}.wd"][:, fpad] == 0)


@pytest.mark.parametrize("policy,mix", [("interleaved", "3way"), ("all-fwd-then-bwd", "3way"),
                                        ("interleaved", "4way"), ("all-fwd-then-bwd", "4way")])
def test_omni_structure_matches_reference(policy, mix):
    """cfg 4 structure: image + audio encoders, backbone, audio decoder; the 4-way mix has
    img+audio samples that take rows from both encoders (parallel-upstream generalisation)."""
    from paper_2605_10501_b200 import graph_workloads as W

    ex = W.omni_executor(tiny=True, mbs_llm=2, mbs_enc=2, lr=0.0, policy=policy, max_pos=2048)
    gb = W.omni_batch(12, seed=5, vocab=W.TINY_LLM.vocab, patch_dim=128, n_codes=W.TINY_DEC.vocab, img_patches=64,
                      frames=40, dec_rows=12, text_lo=16, text_hi=60, mix=mix)
    if mix == "4way":
        assert ((gb.up["image_enc"].rows > 0) & (gb.up["audio_enc"].rows > 0)).any()
    _snapshot(ex)
    st = ex.step(gb)
    _check(ex, gb, st)


def test_policies_give_the_same_step():
    """ExecPolicy changes the stage order only: same loss and gradients."""
    from paper_2605_10501_b200 import graph_workloads as W

    out = []
    for policy in ("interleaved", "all-fwd-then-bwd"):
        ex = W.omni_executor(tiny=True, mbs_llm=2, mbs_enc=2, lr=0.0, policy=policy, max_pos=2048)
        gb = W.omni_batch(12, seed=6, vocab=W.TINY_LLM.vocab, patch_dim=128, n_codes=W.TINY_DEC.vocab,
                          img_patches=64, frames=40, dec_rows=12, text_lo=16, text_hi=60, mix="4way")
        st = ex.step(gb)
        out.append((st.loss, {n: m.p.grad.clone() for n, m in ex.mod.items() if m.trainable}))
        ev = ex.stage_events()
        crit = [nm for nm, _, _ in ev["llm"]]
        if policy == "interleaved":
            assert crit[:2] == ["f_c0", "b_c0"]
        else:
            assert crit[: len(crit) // 2] == [f"f_c{m}" for m in range(len(crit) // 2)]
    assert abs(out[0][0] - out[1][0]) <= 1e-5 * abs(out[0][0])
    for n in out[0][1]:
        assert rel(out[0][1][n], out[1][1][n]) < 1e-4, n


def test_kd_graph_matches_kd_executor():
    """The KD graph on the generic executor == the tuned KDExecutor (same seeds): loss + grads."""
    from paper_2605_10501_b200 import graph_workloads as W
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ids = synthetic_ids(8, 128, 512, seed=8)
    a = KDExecutor(n_gpus=1, batch_per_rank=8, seq=128, mbs=2, teacher="test_tiny", student="test_tiny", lr=0.0,
                   teacher_mbs=4)
    sa = a.step(torch.from_numpy(ids).cuda())
    ex = W.kd_executor(mbs=2, teacher_mbs=4, lr=0.0, seq=128)
    sb = ex.step(W.kd_batch(ids))
    assert abs(sa.loss - sb.loss) <= 1e-3 * abs(sa.loss), (sa.loss, sb.loss)
    assert rel(ex.mod["student"].p.grad, a.student.p.grad) < 2e-2
