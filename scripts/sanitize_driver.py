"""One small launch of each hot kernel family for compute-sanitizer (racecheck / synccheck /
memcheck): attention fwd+bwd at head_dim 64 and 128 (varlen, causal, GQA), the tcgen05 GEMM
(bf16 store, fp32 accumulate, RoPE/SwiGLU/residual epilogues), K9, the K5b handoff index + K6
scatter, and one plan (K1-K5)."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(which):
    from paper_2605_10501_b200 import attention as A
    from paper_2605_10501_b200 import dense, kernels as K
    from paper_2605_10501_b200.transformer import rope_table

    torch.manual_seed(0)
    if which in ("attn", "all"):
        for dh in (64, 128):
            lens = [1, 127, 300]
            H, Hk = 4, 2
            T = sum(lens)
            cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32, device="cuda")
            q = torch.randn(T, H, dh, device="cuda").bfloat16()
            k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
            v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
            o = torch.empty_like(q)
            sc = 1 / math.sqrt(dh)
            plan = A.plan(cu, T)
            lse = A.attn_fwd(q, k, v, cu, 300, True, o, sc, plan=plan)
            do = torch.randn_like(q)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            pos = torch.cat([torch.arange(n, dtype=torch.int32) for n in lens]).cuda()
            cs = rope_table(512, dh, 10000.0, "cuda")
            A.attn_bwd(do, q, k, v, o, lse, cu, 300, True, dq, dk, dv, sc, rope=(pos, cs), plan=plan)
            torch.cuda.synchronize()
    if which in ("gemm", "all"):
        M, N, Kd = 300, 640, 256
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        w = torch.randn(N, Kd, device="cuda").bfloat16()
        dense.linear_fwd(x, w)
        pos = torch.arange(M, dtype=torch.int32, device="cuda")
        dense.linear_fwd_rope(x, w, pos, rope_table(512, 64, 1e4, "cuda"), 512)
        dense.linear_fwd_rope(x, w, pos, rope_table(512, 128, 1e4, "cuda"), 512, head_dim=128)
        s = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        dense.linear_fwd_swiglu(x, w, s)
        dense.linear_fwd_residual(x, w, torch.randn(M, N, device="cuda").bfloat16())
        dw = torch.zeros(N, Kd, device="cuda")
        dense.linear_wgrad(torch.randn(M, N, device="cuda").bfloat16(), x, dw)
        torch.cuda.synchronize()
    if which in ("kd", "all"):
        t = torch.randn(33, 4096, device="cuda").bfloat16()
        st = torch.randn(33, 4096, device="cuda").bfloat16()
        loss = torch.empty(33, device="cuda")
        K.kd_loss(t, st, st, loss, 0.5)
        torch.cuda.synchronize()
    if which in ("handoff", "all"):
        from paper_2605_10501_b200.handoff import handoff_index, scatter_mb

        d = lambda a: torch.tensor(np.asarray(a, dtype=np.int32), device="cuda")  # noqa: E731
        rows = np.array([3, 0, 2, 5])
        ix = handoff_index(d([0, 2, 3]), d([3, 1, 0, 2]), d([0, 9, 16, 26]), 2, d(rows), d([1, 0, 2, 0]), 10, 10)
        buf = torch.randn(10, 64, device="cuda").bfloat16()
        x = torch.zeros(40, 64, device="cuda", dtype=torch.bfloat16)
        scatter_mb(ix, 0, buf, x)
        scatter_mb(ix, 1, buf, x)
        torch.cuda.synchronize()
    if which in ("plan", "all"):
        from paper_2605_10501_b200 import recipes as R
        from paper_2605_10501_b200.costs import cost_table
        from paper_2605_10501_b200.scheduling import DevicePlanner

        rec = R.vlm_tiny(4, 64, 0)
        tab = rec.graph.tables
        tok = np.zeros((len(tab.sub_names), rec.batch), dtype=np.int32)
        for b, n in enumerate(tab.sub_names):
            if n in rec.tokens:
                tok[b] = rec.tokens[n]
        p = DevicePlanner(rec.graph, rec.configs, "interleaved", max_batch=rec.batch)
        p.ids[: rec.batch].copy_(torch.arange(rec.batch, dtype=torch.int32))
        p.plan_tokens(torch.from_numpy(cost_table(rec.graph, rec.configs, rec.params)).cuda(),
                      torch.from_numpy(tok).cuda(), rec.batch)
        torch.cuda.synchronize()
    print("ok", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
