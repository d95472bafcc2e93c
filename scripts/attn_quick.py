"""Our K8 forward/backward TFLOP/s at the head-to-head shapes (same timing as attn_h2h.py, no
library baselines): quick A/B for attention changes.  One JSON line per shape."""
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402
from attn_h2h import SHAPES, timeit  # noqa: E402


def main():
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
        t_f = timeit(lambda: A.attn_fwd(q, k, v, cu, L, causal, o, sc, plan=plan), iters=20)
        lse = A.attn_fwd(q, k, v, cu, L, causal, o, sc, plan=plan)
        do = torch.randn_like(q)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        t_b = timeit(lambda: A.attn_bwd(do, q, k, v, o, lse, cu, L, causal, dq, dk, dv, sc, plan=plan), iters=20)
        print(json.dumps({"shape": label, "fwd_tflops": flops / t_f / 1e12, "bwd_tflops": 2.5 * flops / t_b / 1e12}),
              flush=True)


if __name__ == "__main__":
    main()
