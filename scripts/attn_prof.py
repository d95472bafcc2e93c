"""One forward+backward of the teacher-shaped attention (for ncu captures)."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402

nseq, L, H, Hk, dh = 4, 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 32, int(sys.argv[2]) if len(sys.argv) > 2 else 4, 64
T = nseq * L
cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
q = torch.randn(T, H, dh, device="cuda").bfloat16()
k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
o = torch.empty_like(q)
for _ in range(2):
    lse = A.attn_fwd(q, k, v, cu, L, True, o, 1 / math.sqrt(dh))
    do = torch.randn_like(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    A.attn_bwd(do, q, k, v, o, lse, cu, L, True, dq, dk, dv, 1 / math.sqrt(dh))
torch.cuda.synchronize()
print("ok")
