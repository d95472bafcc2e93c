"""One shape of the tcgen05 GEMM (K7) a few times, for ncu captures.

    python scripts/gemm_prof.py M N K [fwd|swiglu|residual|dgrad|wgrad]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import dense  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "fwd"
a = torch.randn(M, K, device="cuda").bfloat16()
w = torch.randn(N, K, device="cuda").bfloat16()
for _ in range(3):
    if mode == "swiglu":
        s = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        dense.linear_fwd_swiglu(a, w, s)
    elif mode == "swiglu_only":  # forward-only sections: only silu(g) * u is stored
        s = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        dense.linear_fwd_swiglu(a, w, s, store_gu=False)
    elif mode == "residual":
        r = torch.randn(M, N, device="cuda").bfloat16()
        dense.linear_fwd_residual(a, w, r)
    elif mode == "dgrad":
        dy = torch.randn(M, N, device="cuda").bfloat16()
        dense.linear_dgrad(dy, w, wt=w.t().contiguous())
    elif mode == "wgrad":
        dy = torch.randn(M, N, device="cuda").bfloat16()
        dw = torch.zeros(N, K, device="cuda")
        dense.linear_wgrad(dy, a, dw)
    else:
        dense.linear_fwd(a, w)
torch.cuda.synchronize()
print("ok")
