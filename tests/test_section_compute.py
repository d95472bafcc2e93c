"""GPU numerics of the section compute against the plain PyTorch fp32 restatement (oracle/torch_ref.py).

Parity for this part is unpinned by the reference (it has no model code); tolerances are stated
per test.  Model-level checks compare with the bf16-rounding-aware oracle (activations rounded to
bf16 where the kernels store them): relative L2 error <= 1e-2 on outputs and every gradient
(measured 2.6e-3 .. 7.6e-3, profiles/r02_parity_report.json), max-normalised error <= 2e-2, losses
<= 1e-3 relative; single-kernel checks: bf16 outputs ~1e-2, fp32 reductions ~1e-4.
"""

import math

import pytest
import torch

from oracle import torch_ref as R

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


def relnorm(a, b):
    """Relative L2 error ||a - b|| / ||b|| (profiles/r02_parity_report.json: 2.6e-3 .. 7.6e-3 here)."""
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def test_rmsnorm_fwd_bwd():
    from paper_2605_10501_b200 import kernels as K

    torch.manual_seed(0)
    T, d = 300, 768
    x = torch.randn(T, d, device="cuda").bfloat16()
    a = torch.randn(T, d, device="cuda").bfloat16()
    w = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    h, y = torch.empty_like(x), torch.empty_like(x)
    r = torch.empty(T, device="cuda")
    K.add_rmsnorm(x, a, h, y, w, r, 1e-5)
    href = (x.float() + a.float()).bfloat16().float()
    assert torch.equal(h, href.bfloat16())
    assert rel(y, R.rms_norm(href, w.float(), 1e-5)) < 1e-2
    # backward vs autograd
    hh = href.clone().requires_grad_(True)
    ww = w.float().clone().requires_grad_(True)
    yr = R.rms_norm(hh, ww, 1e-5)
    dy = torch.randn(T, d, device="cuda").bfloat16()
    dres = torch.randn(T, d, device="cuda").bfloat16()
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    dw = torch.zeros(d, device="cuda")
    K.rmsnorm_bwd(dy, h, w, r, dres, dx, dw)
    assert rel(dx, hh.grad + dres.float()) < 1e-2
    assert rel(dw, ww.grad) < 1e-3


def test_swiglu_rope_embed():
    from paper_2605_10501_b200 import kernels as K
    from paper_2605_10501_b200.transformer import rope_table

    torch.manual_seed(1)
    T, F = 257, 512
    gu = torch.randn(T, 2 * F, device="cuda").bfloat16()
    out = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
    K.swiglu(gu, out)
    gi = R.gate_index(F, "cuda")  # interleaved [g(32) | u(32)] blocks
    g, u = gu.float()[:, gi].requires_grad_(True), gu.float()[:, gi + 32].requires_grad_(True)
    ref = torch.nn.functional.silu(g) * u
    assert rel(out, ref) < 1e-2
    dout = torch.randn(T, F, device="cuda").bfloat16()
    ref.backward(dout.float())
    dgu = torch.empty_like(gu)
    K.swiglu_bwd(dout, gu, dgu)
    assert rel(dgu[:, gi], g.grad) < 2e-2 and rel(dgu[:, gi + 32], u.grad) < 2e-2
    # RoPE fwd then bwd is the identity (orthogonal rotation), and matches the fp32 formula
    H, dh = 6, 64
    x = torch.randn(T, H * dh + 32, device="cuda").bfloat16()  # row pitch > H*dh
    pos = torch.randint(0, 2048, (T,), device="cuda", dtype=torch.int32)
    cs = rope_table(2048, dh, 10000.0, "cuda")
    y = x.clone()
    K.rope(y[:, : H * dh], pos, cs, H, dh)
    ref = R.rope(x[:, : H * dh].float().view(T, H, dh), pos, 10000.0).view(T, H * dh)
    assert rel(y[:, : H * dh], ref) < 1e-2
    assert torch.equal(y[:, H * dh:], x[:, H * dh:])
    K.rope(y[:, : H * dh], pos, cs, H, dh, backward=True)
    assert rel(y, x) < 2e-2
    # embedding gather / scatter-add
    V, d = 1000, 128
    table = torch.randn(V, d, device="cuda").bfloat16()
    ids = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    e = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    K.embed(table, ids, e)
    assert torch.equal(e, table[ids.long()])
    dtab = torch.zeros(V, d, device="cuda")
    K.embed_bwd(e, ids, dtab)
    ref = torch.zeros(V, d, device="cuda").index_add_(0, ids.long(), e.float())
    assert rel(dtab, ref) < 1e-5


def test_adamw_matches_reference():
    from paper_2605_10501_b200 import kernels as K

    torch.manual_seed(2)
    n = 4096
    p, g = torch.randn(n, device="cuda"), torch.randn(n, device="cuda")
    m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    pb = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    pr, mr, vr = p.clone(), m.clone(), v.clone()
    for step in (1, 2, 3):
        K.adamw(p, g, m, v, pb, 1e-3, step)
        R.adamw_reference(pr, g, mr, vr, 1e-3, step)
    assert rel(p, pr) < 1e-6 and torch.equal(pb, p.bfloat16())


@pytest.mark.parametrize("T,V", [(64, 32000), (33, 128256 // 8 * 8), (8, 64), (300, 40000), (5, 150000), (3, 4104)])
def test_kd_loss_fused(T, V):
    from paper_2605_10501_b200 import kernels as K

    torch.manual_seed(T)
    t = (3 * torch.randn(T, V, device="cuda")).bfloat16()
    s = (3 * torch.randn(T, V, device="cuda")).bfloat16()
    ss = s.float().clone().requires_grad_(True)
    ref = R.kd_loss(t.float(), ss)
    (ref.sum() * 0.5).backward()
    loss = torch.empty(T, device="cuda")
    ds = torch.empty_like(s)
    K.kd_loss(t, s, ds, loss, grad_scale=0.5)
    assert rel(loss, ref) < 1e-4  # fp32 reductions
    assert rel(ds, ss.grad) < 1e-2  # bf16 output
    # in-place (ds aliases the student logits)
    s2 = s.clone()
    K.kd_loss(t, s2, s2, loss, grad_scale=0.5)
    assert torch.equal(s2, ds)
    # loss only (no gradient)
    loss2 = torch.empty(T, device="cuda")
    K.kd_loss(t, s, None, loss2, grad_scale=0.5)
    assert torch.equal(loss2, loss)


@pytest.mark.parametrize("T,V", [(64, 32000), (37, 152064), (9, 64), (130, 32768)])
def test_ce_loss_fused(T, V):
    """Next-token CE with ignore index (label < 0) vs torch fp32 cross_entropy: loss per row and
    ds = grad_scale * (softmax - onehot), in place over the logits."""
    from paper_2605_10501_b200 import kernels as K

    torch.manual_seed(V + T)
    s = (3 * torch.randn(T, V, device="cuda")).bfloat16()
    lab = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    lab[::7] = -1
    ss = s.float().clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(ss, lab.long().clamp_min(0), reduction="none") * (lab >= 0)
    (ref.sum() * 0.5).backward()
    loss = torch.empty(T, device="cuda")
    ds = s.clone()
    K.ce_loss(ds, lab, ds, loss, 0.5)
    assert rel(loss, ref) < 1e-4
    assert rel(ds, ss.grad) < 1e-2
    assert torch.all(ds[lab < 0] == 0) and torch.all(loss[lab < 0] == 0)


def _tiny_model(seed=0, shape_name="test_tiny"):
    from paper_2605_10501_b200.transformer import SHAPES, FlatParams, Transformer

    shape = SHAPES[shape_name]
    p = FlatParams(shape.param_shapes(), torch.device("cuda"), trainable=True, seed=seed)
    return shape, Transformer(shape, p, torch.device("cuda"), max_pos=1024)


@pytest.mark.parametrize("shape_name", ["test_tiny", "test_tiny_hd128"])
@pytest.mark.parametrize("causal", [True, False])
def test_transformer_fwd_bwd_vs_fp32(causal, shape_name):
    import dataclasses

    from paper_2605_10501_b200 import kernels as K
    from paper_2605_10501_b200.transformer import Batch, SHAPES, FlatParams, Transformer

    shape = dataclasses.replace(SHAPES[shape_name], causal=causal)
    p = FlatParams(shape.param_shapes(), torch.device("cuda"), trainable=True, seed=3)
    model = Transformer(shape, p, torch.device("cuda"), max_pos=1024)
    lens = [100, 37, 256, 1]
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
    T = sum(lens)
    ids = torch.randint(0, shape.vocab, (T,), device="cuda", dtype=torch.int32)
    pos = torch.empty(T, dtype=torch.int32, device="cuda")
    K.positions(cu, len(lens), pos)
    b = Batch(ids, cu, pos, max(lens))
    yf, ctx = model.forward(b)
    logits = model.logits(yf)
    flat = p.w.float().clone().requires_grad_(True)
    P = R.param_views(shape, flat)
    yr = R.forward(shape, P, ids, cu, bf16=True)  # rounding-aware oracle (bf16 at the kernels' store points)
    lr_ = R.rb(yr @ R.head_weight(shape, P).t())
    assert rel(yf, yr) < 2e-2 and relnorm(yf, yr) < 1e-2
    assert rel(logits, lr_) < 2e-2 and relnorm(logits, lr_) < 1e-2
    dl = (torch.randn_like(lr_) * 0.01).bfloat16()
    lr_.backward(dl.float())
    p.zero_grad()
    model.backward(ctx, dlogits=dl)
    for name in ("embed", "head", "lnf", "l1.wd", "l1.wgu", "l0.wqkv", "l0.wo", "l0.ln1"):
        got, want = p.g(name), R.param_views(shape, flat.grad)[name]
        assert rel(got, want) < 2e-2 and relnorm(got, want) < 1e-2, name


def test_kd_executor_step_matches_reference():
    """One co-resident KD step on tiny shapes == fp32 autograd restatement (loss + grads)."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ex = KDExecutor(n_gpus=1, batch_per_rank=4, seq=128, mbs=2, teacher="test_tiny", student="test_tiny", lr=0.0)
    ids = torch.from_numpy(synthetic_ids(4, 128, 512, seed=5)).cuda()
    t_flat = ex.teacher.p.w.float()
    s_flat = ex.student.p.w.float()
    st = ex.step(ids)
    cu = torch.arange(0, 4 * 128 + 1, 128, dtype=torch.int32, device="cuda")
    tok, grad = R.kd_step_reference(ex.tshape, ex.sshape, t_flat, s_flat, ex.t_head.float(), ids.reshape(-1), cu,
                                    global_tokens=4 * 128, bf16=True)
    ref_loss = tok.sum().item() / (4 * 128)
    assert abs(st.loss - ref_loss) / max(abs(ref_loss), 1e-6) < 1e-3  # measured 4e-5
    got = R.param_views(ex.sshape, ex.student.p.grad)
    want = R.param_views(ex.sshape, grad)
    assert relnorm(ex.student.p.grad, grad) < 1e-2  # measured 2.6e-3
    for name in ("embed", "lnf", "l0.wqkv", "l1.wd"):
        assert rel(got[name], want[name]) < 2e-2 and relnorm(got[name], want[name]) < 1e-2, name
    assert 0.0 <= st.stall_frac <= 1.0


@pytest.mark.parametrize("d", [192, 768, 2048, 4096])
def test_rmsnorm_all_widths(d):
    """Register-resident fast path (multiples of 256) and the generic path agree with fp32."""
    from paper_2605_10501_b200 import kernels as K

    torch.manual_seed(d)
    T = 333
    x = torch.randn(T, d, device="cuda").bfloat16()
    a = torch.randn(T, d, device="cuda").bfloat16()
    w = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    h, y = torch.empty_like(x), torch.empty_like(x)
    r = torch.empty(T, device="cuda")
    K.add_rmsnorm(x, a, h, y, w, r, 1e-5)
    href = (x.float() + a.float()).bfloat16().float()
    assert torch.equal(h, href.bfloat16())
    assert rel(y, R.rms_norm(href, w.float(), 1e-5)) < 1e-2
    hh = href.clone().requires_grad_(True)
    ww = w.float().clone().requires_grad_(True)
    dy = torch.randn(T, d, device="cuda").bfloat16()
    R.rms_norm(hh, ww, 1e-5).backward(dy.float())
    dx, dw = torch.empty_like(x), torch.zeros(d, device="cuda")
    K.rmsnorm_bwd(dy, h, w, r, None, dx, dw)
    assert rel(dx, hh.grad) < 1e-2 and rel(dw, ww.grad) < 1e-3


def test_measured_trace_and_model_crosscheck(tmp_path):
    """Device stage timestamps -> simulator StageEvents -> chrome trace; model re-run."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids
    from paper_2605_10501_b200.simulator import export_trace

    ex = KDExecutor(n_gpus=1, batch_per_rank=8, seq=128, mbs=2, teacher="test_tiny", student="test_tiny")
    ids = torch.from_numpy(synthetic_ids(8, 128, 512, seed=6)).cuda()
    ex.step(ids)
    ev = ex.measured_events()
    assert {e.phase for e in ev} == {"f_bc", "f_c", "b_c"} and len(ev) == 3 * 4
    assert all(e.end >= e.start >= 0 for e in ev)
    export_trace(ev, str(tmp_path / "trace.json"))
    mk, cidle, span, midle = ex.crosscheck()
    assert mk > 0 and cidle >= 0 and span > 0 and midle >= -1e-9


def test_kd_teacher_micro_batch_size_is_a_schedule_knob():
    """SectionConfig.mbs per section: a teacher micro-batch twice the student's gives the same step
    (loss, student gradients) -- only GEMM tiling / reduction order differ."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ids = torch.from_numpy(synthetic_ids(8, 128, 512, seed=7)).cuda()
    res = []
    for tm in (2, 4):
        ex = KDExecutor(n_gpus=1, batch_per_rank=8, seq=128, mbs=2, teacher="test_tiny", student="test_tiny",
                        lr=0.0, teacher_mbs=tm)
        st = ex.step(ids)
        res.append((st.loss, ex.student.p.grad.clone()))
        ev = ex.measured_events()
        assert sorted(e.sample_id for e in ev if e.phase == "f_bc") == list(range(4))
    assert abs(res[0][0] - res[1][0]) / abs(res[0][0]) < 1e-3
    g0, g1 = res[0][1], res[1][1]
    assert ((g0 - g1).abs().max() / g0.abs().max()).item() < 2e-2


def test_kd_uneven_batch_and_micro_batch_ratio():
    """10 samples, student micro-batches of 4 and teacher micro-batches of 8: partial last micro-
    batches on both sides, and a partial teacher micro-batch feeding a partial student one -- same
    step as equal micro-batches."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ids = torch.from_numpy(synthetic_ids(10, 128, 512, seed=9)).cuda()
    res = []
    for tm in (4, 8):
        ex = KDExecutor(n_gpus=1, batch_per_rank=10, seq=128, mbs=4, teacher="test_tiny", student="test_tiny",
                        lr=0.0, teacher_mbs=tm)
        st = ex.step(ids)
        assert math.isfinite(st.loss)
        res.append((st.loss, ex.student.p.grad.clone()))
    assert abs(res[0][0] - res[1][0]) / abs(res[0][0]) < 1e-3
    assert ((res[0][1] - res[1][1]).abs().max() / res[0][1].abs().max()).item() < 2e-2


def test_kd_plan_ahead_matches_synchronous_plan():
    """step(plan_ahead=True) builds the next schedule beside the current step: same losses and
    gradients as planning at the start of every step; the plan's device time is still reported."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ids = torch.from_numpy(synthetic_ids(8, 128, 512, seed=9)).cuda()
    out = []
    for ahead in (False, True):
        ex = KDExecutor(n_gpus=1, batch_per_rank=8, seq=128, mbs=2, teacher="test_tiny", student="test_tiny",
                        lr=1e-3)
        losses = [ex.step(ids, plan_ahead=ahead) for _ in range(3)]
        out.append(([s.loss for s in losses], ex.student.p.grad.clone(), losses[-1].plan_ms))
    # split-K weight gradients are reduce-added in L2 (order not fixed): fp32-rounding tolerance
    assert all(abs(a - b) <= 1e-6 * abs(a) for a, b in zip(out[0][0], out[1][0]))
    assert ((out[0][1] - out[1][1]).abs().max() / out[0][1].abs().max()).item() < 1e-5
    assert out[1][2] > 0


def test_kd_executor_hd128_teacher_matches_reference():
    """KD step with a head_dim-128 GQA teacher (the cfg 5 teacher's attention / RoPE shape) ==
    fp32 autograd restatement (loss + student grads)."""
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids

    ex = KDExecutor(n_gpus=1, batch_per_rank=4, seq=256, mbs=2, teacher="test_tiny_hd128", student="test_tiny",
                    lr=0.0)
    ids = torch.from_numpy(synthetic_ids(4, 256, 512, seed=15)).cuda()
    t_flat = ex.teacher.p.w.float()
    s_flat = ex.student.p.w.float()
    st = ex.step(ids)
    cu = torch.arange(0, 4 * 256 + 1, 256, dtype=torch.int32, device="cuda")
    tok, grad = R.kd_step_reference(ex.tshape, ex.sshape, t_flat, s_flat, ex.t_head.float(), ids.reshape(-1), cu,
                                    global_tokens=4 * 256, bf16=True)
    ref_loss = tok.sum().item() / (4 * 256)
    assert abs(st.loss - ref_loss) / max(abs(ref_loss), 1e-6) < 1e-3
    got = R.param_views(ex.sshape, ex.student.p.grad)
    want = R.param_views(ex.sshape, grad)
    assert relnorm(ex.student.p.grad, grad) < 1e-2
    for name in ("embed", "lnf", "l0.wqkv", "l1.wd"):
        assert rel(got[name], want[name]) < 2e-2 and relnorm(got[name], want[name]) < 1e-2, name
