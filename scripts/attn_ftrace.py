"""Diag-only: forward pipeline timeline of CTA 0 per item (lib built from scripts/diag/make_ftrace.py)."""
import ctypes
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import _native, attention as A  # noqa: E402

nseq, L, H, Hk = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 2048, 32, 4)))
T, dh = nseq * L, 64
cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(T, h, dh, device="cuda").bfloat16() for h in (H, Hk, Hk))
o = torch.empty_like(q)
for _ in range(3):
    A.attn_fwd(q, k, v, cu, L, True, o, 1 / math.sqrt(dh))
torch.cuda.synchronize()
buf = np.zeros((20, 1024), dtype=np.int64)
assert _native.lib().maestro_diag_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
n_items = int((buf[6] > 0).sum())
n_tiles = int((buf[1] > 0).sum())
t0 = buf[6][0]
print("items", n_items, "tiles", n_tiles)
g = 0
tile_t = []
for j in range(n_items):
    nk = int(buf[7][j])
    start = buf[6][j] - t0
    waits = [int(buf[1][g + i] - buf[0][g + i]) for i in range(nk)]
    work = [int(buf[2][g + i] - buf[1][g + i]) for i in range(nk)]
    epi = int(buf[4][j] - buf[3][j]) if buf[3][j] else -1
    dur = int(buf[6][j + 1] - buf[6][j]) if j + 1 < n_items else -1
    print(f"item {j:3d} n_kv {nk:3d} start {start:9d} dur {dur:7d} per-tile {dur / max(nk, 1):7.0f}  epi {epi:6d}  "
          f"s_wait sum {sum(waits):6d} (first {waits[0]:5d})  work med {int(np.median(work)):5d} first {work[0]:5d} last {work[-1]:5d}")
    g += nk
