"""Bidirectional head_dim-64 attention forward at the encoder shapes (cfg 1 ViT-tiny: 32 x 196
tokens, 3 heads; cfg 4 audio encoder: 8 x 1500, 20 heads; 16 x 375 packed), our kernel only, TFLOP/s."""
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402
from attn_h2h import timeit  # noqa: E402

for label, B, L, H in (("vit-tiny", 32, 196, 3), ("audio-enc", 8, 1500, 20), ("audio-375", 16, 375, 20)):
    T = B * L
    cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
    q, k, v = (torch.randn(T, H, 64, device="cuda").bfloat16() for _ in range(3))
    o = torch.empty_like(q)
    plan = A.plan(cu, T)
    t = timeit(lambda: A.attn_fwd(q, k, v, cu, L, False, o, 0.125, plan=plan), iters=50)
    print(json.dumps({"shape": label, "fwd_tflops": 4 * B * L * L * 64 * H / t / 1e12, "us": t * 1e6}), flush=True)
