"""Microbenchmark: tcgen05 varlen attention (K8) vs the flash-attn 2 library on B200."""

import json
import math
import sys
from pathlib import Path

import torch

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


def main():
    from flash_attn import flash_attn_interface as fa

    out = []
    for nseq, L, H, Hk in [(4, 2048, 32, 4), (4, 2048, 12, 12), (2, 8192, 32, 8), (16, 196, 3, 3)]:
        causal = L != 196
        T = nseq * L
        dh = 64
        cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
        q = torch.randn(T, H, dh, device="cuda").bfloat16()
        k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
        v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
        o = torch.empty_like(q)
        sc = 1 / math.sqrt(dh)
        flops = 4 * nseq * L * L * dh * H * (0.5 if causal else 1.0)
        t_f = timeit(lambda: A.attn_fwd(q, k, v, cu, L, causal, o, sc))
        lse = A.attn_fwd(q, k, v, cu, L, causal, o, sc)
        do = torch.randn_like(q)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        t_b = timeit(lambda: A.attn_bwd(do, q, k, v, o, lse, cu, L, causal, dq, dk, dv, sc))
        t_ff = timeit(lambda: fa._flash_attn_varlen_forward(q, k, v, cu, cu, L, L, 0.0, sc, causal))
        o2, lse2, _, _ = fa._flash_attn_varlen_forward(q, k, v, cu, cu, L, L, 0.0, sc, causal)
        t_fb = timeit(lambda: fa._flash_attn_varlen_backward(do, q, k, v, o2, lse2, dq, dk, dv, cu, cu, L, L, 0.0, sc,
                                                             causal, -1, -1, 0.0, None, False))
        rec = {"nseq": nseq, "L": L, "H": H, "Hk": Hk, "causal": causal,
               "fwd_tflops": flops / t_f / 1e12, "bwd_tflops": 2.5 * flops / t_b / 1e12,
               "fa2_fwd_tflops": flops / t_ff / 1e12, "fa2_bwd_tflops": 2.5 * flops / t_fb / 1e12}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/attn_bench.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
