"""Head-to-head: tcgen05 varlen attention (K8) vs cuDNN's sm100 SDPA (torch SDPA, cuDNN backend)
and flash-attn 2.8 on the same B200, at the KD / cfg 3 / cfg 5 shapes (head_dim 64 and 128).

Sequences of equal length (cuDNN SDPA takes dense [B, H, L, dh]); our kernel runs them packed
(cu_seqlens).  TFLOP/s = 4 * B * L^2 * dh * H (x 1/2 causal) / time; backward = 2.5x forward's
FLOPs.  Writes gpurun_out/attn_h2h.json.
"""

import json
import math
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


SHAPES = [  # (label, B, L, H, Hk, dh, causal)
    ("kd teacher 1.1B", 4, 2048, 32, 4, 64, True),
    ("kd student 125M", 8, 2048, 12, 12, 64, True),
    ("cfg5 teacher 8B", 2, 8192, 32, 8, 128, True),
    ("cfg5 student 1B", 1, 8192, 32, 8, 64, True),
    ("cfg3 backbone 7B", 2, 4096, 28, 4, 128, True),
    ("cfg3 ViT (hd 80 padded to 128)", 4, 4096, 16, 16, 128, False),
]


def main():
    out = []
    try:
        from flash_attn import flash_attn_interface as fa
    except Exception:  # noqa: BLE001
        fa = None
    for label, B, L, H, Hk, dh, causal in SHAPES:
        T = B * L
        cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
        q = torch.randn(T, H, dh, device="cuda").bfloat16()
        k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
        v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
        o = torch.empty_like(q)
        sc = 1 / math.sqrt(dh)
        flops = 4 * B * L * L * dh * H * (0.5 if causal else 1.0)
        plan = A.plan(cu, T)
        t_f = timeit(lambda: A.attn_fwd(q, k, v, cu, L, causal, o, sc, plan=plan))
        lse = A.attn_fwd(q, k, v, cu, L, causal, o, sc, plan=plan)
        do = torch.randn_like(q)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        t_b = timeit(lambda: A.attn_bwd(do, q, k, v, o, lse, cu, L, causal, dq, dk, dv, sc, plan=plan))
        rec = {"shape": label, "B": B, "L": L, "H": H, "Hk": Hk, "dh": dh, "causal": causal,
               "ours_fwd_tflops": flops / t_f / 1e12, "ours_bwd_tflops": 2.5 * flops / t_b / 1e12}
        # cuDNN SDPA (dense, GQA expanded: the cuDNN backend wants equal head counts)
        qd = q.view(B, L, H, dh).transpose(1, 2).contiguous().requires_grad_(True)
        kd = k.view(B, L, Hk, dh).repeat_interleave(H // Hk, 2).transpose(1, 2).contiguous().requires_grad_(True)
        vd = v.view(B, L, Hk, dh).repeat_interleave(H // Hk, 2).transpose(1, 2).contiguous().requires_grad_(True)
        dod = do.view(B, L, H, dh).transpose(1, 2).contiguous()
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel

            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                t_cf = timeit(lambda: F.scaled_dot_product_attention(qd, kd, vd, is_causal=causal, scale=sc))
                od = F.scaled_dot_product_attention(qd, kd, vd, is_causal=causal, scale=sc)
                t_cb = timeit(lambda: torch.autograd.grad(od, (qd, kd, vd), dod, retain_graph=True))
            rec["cudnn_fwd_tflops"] = flops / t_cf / 1e12
            rec["cudnn_bwd_tflops"] = 2.5 * flops / t_cb / 1e12
        except Exception as exc:  # noqa: BLE001
            rec["cudnn_error"] = repr(exc)[:200]
        if fa is not None:
            try:
                t_ff = timeit(lambda: fa._flash_attn_varlen_forward(q, k, v, cu, cu, L, L, 0.0, sc, causal))
                o2, lse2, _, _ = fa._flash_attn_varlen_forward(q, k, v, cu, cu, L, L, 0.0, sc, causal)
                t_fb = timeit(lambda: fa._flash_attn_varlen_backward(do, q, k, v, o2, lse2, dq, dk, dv, cu, cu, L, L,
                                                                     0.0, sc, causal, -1, -1, 0.0, None, False))
                rec["fa2_fwd_tflops"] = flops / t_ff / 1e12
                rec["fa2_bwd_tflops"] = 2.5 * flops / t_fb / 1e12
            except Exception as exc:  # noqa: BLE001
                rec["fa2_error"] = repr(exc)[:200]
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del qd, kd, vd, dod
        torch.cuda.empty_cache()
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/attn_h2h.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
