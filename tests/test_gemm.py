"""GPU numerics of the tcgen05 GEMM (K7) against a plain PyTorch fp32 reference.

Tolerance: operands are bf16; accumulation is fp32 in TMEM.  fp32 outputs must match an
fp32 reference of the same bf16 operands to 1e-4 relative (sum-order differences only);
bf16 outputs to one bf16 ulp-ish (2^-7 relative of max magnitude).
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (300, 264, 200), (1000, 768, 768), (2048, 2048, 2048), (129, 8, 1000), (4096, 5632, 2048)]


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_fwd(M, N, K):
    from paper_2605_10501_b200 import dense

    torch.manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    ref = x.float() @ w.float().t()
    y = dense.linear_fwd(x, w)
    assert _rel(y, ref) < 8e-3
    y32 = torch.empty(M, N, device="cuda")
    dense.gemm(x, w, y32, M, N, K, False, False, dense.EPI_F32)
    assert _rel(y32, ref) < 1e-4


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_dgrad(M, N, K):
    from paper_2605_10501_b200 import dense

    torch.manual_seed(1 + M)
    dy = torch.randn(M, N, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    if K % 8:
        pytest.skip("K must be a multiple of 8")
    ref = dy.float() @ w.float()
    dx = dense.linear_dgrad(dy, w)
    assert _rel(dx, ref) < 8e-3


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_wgrad_accumulate(M, N, K):
    from paper_2605_10501_b200 import dense

    torch.manual_seed(2 + N)
    if M % 8 or K % 8:
        pytest.skip("alignment")
    dy = torch.randn(M, N, device="cuda").bfloat16()
    x = torch.randn(M, K, device="cuda").bfloat16()
    dw = torch.randn(N, K, device="cuda")
    ref = dw + dy.float().t() @ x.float()
    dense.linear_wgrad(dy, x, dw, accumulate=True)
    assert _rel(dw, ref) < 1e-4


def test_strided_views():
    """Operands that are column slices of wider buffers (fused QKV layouts)."""
    from paper_2605_10501_b200 import dense

    torch.manual_seed(7)
    big = torch.randn(512, 3 * 256, device="cuda").bfloat16()
    x = big[:, 256:512]
    w = torch.randn(384, 256, device="cuda").bfloat16()
    out = torch.empty(512, 384, device="cuda", dtype=torch.bfloat16)
    dense.gemm(x, w, out, 512, 384, 256, False, False, dense.EPI_BF16, lda=big.stride(0))
    assert _rel(out, x.float() @ w.float().t()) < 8e-3


@pytest.mark.parametrize("M,N,K", [(8192, 768, 768), (8192, 2304, 768), (8192, 768, 3072), (8192, 6144, 768)])
def test_training_shapes_all_paths(M, N, K):
    """Student-layer shapes: BN=128 wave-quantisation path (fwd) and split-K atomic wgrad."""
    from paper_2605_10501_b200 import dense

    torch.manual_seed(M + N)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    assert _rel(dense.linear_fwd(x, w), x.float() @ w.float().t()) < 8e-3
    dy = torch.randn(M, N, device="cuda").bfloat16()
    assert _rel(dense.linear_dgrad(dy, w), dy.float() @ w.float()) < 8e-3
    dw = torch.randn(N, K, device="cuda")
    ref = dw + dy.float().t() @ x.float()
    dense.linear_wgrad(dy, x, dw)
    assert _rel(dw, ref) < 1e-4


def test_fused_epilogues_rope_swiglu():
    """RoPE and SwiGLU fused into the 2-CTA GEMM epilogue == unfused fp32 formulas."""
    from oracle import torch_ref as R
    from paper_2605_10501_b200 import dense
    from paper_2605_10501_b200.transformer import rope_table

    torch.manual_seed(11)
    T, K, H = 1000, 512, 6
    x = torch.randn(T, K, device="cuda").bfloat16()
    w = torch.randn(H * 64 + 128, K, device="cuda").bfloat16()  # 6 rotated heads + 2 plain
    pos = torch.randint(0, 1024, (T,), device="cuda", dtype=torch.int32)
    cs = rope_table(1024, 64, 10000.0, "cuda")
    y = dense.linear_fwd_rope(x, w, pos, cs, H * 64)
    ref = x.float() @ w.float().t()
    rot = R.rope(ref[:, : H * 64].view(T, H, 64), pos, 10000.0).view(T, H * 64)
    assert _rel(y[:, : H * 64], rot) < 1e-2 and _rel(y[:, H * 64:], ref[:, H * 64:]) < 8e-3
    F = 384
    wgu = torch.randn(2 * F, K, device="cuda").bfloat16()
    s = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
    gu = dense.linear_fwd_swiglu(x, wgu, s)
    gref = x.float() @ wgu.float().t()
    assert _rel(gu, gref) < 8e-3
    gi = R.gate_index(F, "cuda")
    sref = torch.nn.functional.silu(gref[:, gi]) * gref[:, gi + 32]
    assert _rel(s, sref) < 2e-2


@pytest.mark.parametrize("M,N,K", [(8192, 768, 768), (8192, 768, 3072), (1000, 768, 2304), (520, 200, 96)])
@pytest.mark.parametrize("bn", ["auto", "192"])
def test_k_major_dgrad_and_192_tiles(M, N, K, bn, monkeypatch):
    """dgrad through the transposed (K-major) weight copy; 256 x 192 CTA-pair tiles (auto choice
    for 768-wide outputs, forced for the other shapes incl. ragged M/N)."""
    from paper_2605_10501_b200 import dense, kernels

    if bn != "auto":
        monkeypatch.setenv("MAESTRO_GEMM_BN", bn)
    torch.manual_seed(M + 3 * N + K)
    w = torch.randn(K, N, device="cuda").bfloat16()  # layer weight [out=K, in=N]
    wt = torch.empty(N, K, device="cuda", dtype=torch.bfloat16)
    kernels.transpose(w, wt)
    torch.cuda.synchronize()
    assert torch.equal(wt, w.t())
    dy = torch.randn(M, K, device="cuda").bfloat16()
    ref = dy.float() @ w.float()
    assert _rel(dense.linear_dgrad(dy, w, wt=wt), ref) < 8e-3
    x = torch.randn(M, K, device="cuda").bfloat16()
    assert _rel(dense.linear_fwd(x, wt), x.float() @ w.float()) < 8e-3
    acc = torch.randn(M, N, device="cuda")
    ref2 = acc + x.float() @ w.float()
    dense.gemm(x, wt, acc, M, N, K, False, False, dense.EPI_F32_ACC)
    assert _rel(acc, ref2) < 1e-4


def test_transpose_ragged():
    from paper_2605_10501_b200 import kernels

    src = torch.randn(200, 72, device="cuda").bfloat16()
    dst = torch.zeros(72, 200, device="cuda", dtype=torch.bfloat16)
    kernels.transpose(src, dst)
    torch.cuda.synchronize()
    assert torch.equal(dst, src.t())


def test_transpose_batched_mixed_shapes():
    from paper_2605_10501_b200 import kernels

    shapes = [(200, 72), (64, 64), (768, 3072), (8, 8), (136, 1000)]
    srcs = [torch.randn(r, c, device="cuda").bfloat16() for r, c in shapes]
    dsts = [torch.zeros(c, r, device="cuda", dtype=torch.bfloat16) for r, c in shapes]
    desc, tiles = kernels.transpose_batch_desc(list(zip(srcs, dsts)), "cuda")
    kernels.transpose_batched(desc, tiles)
    torch.cuda.synchronize()
    for s_, d_ in zip(srcs, dsts):
        assert torch.equal(d_, s_.t())


@pytest.mark.parametrize("M,N,K", [(8192, 2048, 2048), (8192, 768, 3072), (1000, 200, 96), (300, 2048, 5632)])
def test_residual_epilogue(M, N, K):
    """h = R + A B^T with the add in the epilogue: fp32 sum rounded once (vs fp32 reference)."""
    from paper_2605_10501_b200 import dense

    torch.manual_seed(M + N + 5)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    big = torch.randn(M, N + 64, device="cuda").bfloat16()  # residual as a strided view
    r = big[:, 32: 32 + N]
    h = dense.linear_fwd_residual(x, w, r)
    ref = r.float() + x.float() @ w.float().t()
    assert _rel(h, ref) < 8e-3


@pytest.mark.parametrize("T,F,K", [(1000, 384, 512), (8192, 2816, 2048)])
def test_swiglu_without_gu_store(T, F, K):
    """Forward-only sections: the gate/up GEMM writes only silu(g) * u (C = NULL)."""
    from oracle import torch_ref as R
    from paper_2605_10501_b200 import dense

    torch.manual_seed(T + F)
    x = torch.randn(T, K, device="cuda").bfloat16()
    wgu = (torch.randn(2 * F, K, device="cuda") * 0.05).bfloat16()
    s = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
    assert dense.linear_fwd_swiglu(x, wgu, s, store_gu=False) is None
    gref = x.float() @ wgu.float().t()
    gi = R.gate_index(F, "cuda")
    sref = torch.nn.functional.silu(gref[:, gi]) * gref[:, gi + 32]
    assert _rel(s, sref) < 2e-2


def test_rope_epilogue_hd128():
    """RoPE over 128-wide heads (pairs (i, i+64), 64 frequencies) in the GEMM epilogue."""
    from oracle import torch_ref as R
    from paper_2605_10501_b200 import dense
    from paper_2605_10501_b200.transformer import rope_table

    torch.manual_seed(12)
    for T, H in ((1000, 5), (4096, 12)):
        K = 1024
        x = torch.randn(T, K, device="cuda").bfloat16()
        w = torch.randn(H * 128 + 256, K, device="cuda").bfloat16()
        pos = torch.randint(0, 8192, (T,), device="cuda", dtype=torch.int32)
        cs = rope_table(8192, 128, 500000.0, "cuda")
        y = dense.linear_fwd_rope(x, w, pos, cs, H * 128, head_dim=128)
        ref = x.float() @ w.float().t()
        rot = R.rope(ref[:, : H * 128].view(T, H, 128), pos, 500000.0).view(T, H * 128)
        assert _rel(y[:, : H * 128], rot) < 1e-2 and _rel(y[:, H * 128:], ref[:, H * 128:]) < 8e-3
