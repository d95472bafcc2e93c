"""One attention call at a named shape (for ncu): python scripts/attn_one.py <shape> [fwd|bwd]."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402

SHAPES = {"kd_teacher": (4, 2048, 32, 4, 64, True), "kd_student": (8, 2048, 12, 12, 64, True),
          "cfg5_teacher": (2, 8192, 32, 8, 128, True), "vit": (4, 4096, 16, 16, 128, False)}


def main():
    B, L, H, Hk, dh, causal = SHAPES[sys.argv[1]]
    mode = sys.argv[2] if len(sys.argv) > 2 else "fwd"
    T = B * L
    cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
    torch.manual_seed(0)
    q = torch.randn(T, H, dh, device="cuda").bfloat16()
    k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    o = torch.empty_like(q)
    plan = A.plan(cu, T)
    sc = 1 / math.sqrt(dh)
    for _ in range(3):
        lse = A.attn_fwd(q, k, v, cu, L, causal, o, sc, plan=plan)
        if mode == "bwd":
            do = torch.randn_like(q)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            A.attn_bwd(do, q, k, v, o, lse, cu, L, causal, dq, dk, dv, sc, plan=plan)
    torch.cuda.synchronize()
    print("ok", sys.argv[1:])


if __name__ == "__main__":
    main()
