"""Diag-only: per-tile pipeline timeline of attention-forward CTA 0 (needs a lib built with the
trace hooks exporting maestro_diag_trace).  Prints clock deltas per KV tile."""
import ctypes
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import _native, attention as A  # noqa: E402

nseq, L, H, Hk = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (2, 8192, 32, 8)))
T, dh = nseq * L, 64
cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
q = torch.randn(T, H, dh, device="cuda").bfloat16()
k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
o = torch.empty_like(q)
for _ in range(3):
    A.attn_fwd(q, k, v, cu, L, True, o, 1 / math.sqrt(dh))
torch.cuda.synchronize()
buf = np.zeros((20, 1024), dtype=np.int64)
assert _native.lib().maestro_diag_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["S_issued", "PV_pfull_seen", "PV_issued", "sm_wait_s", "sm_s_full", "sm_ldtm_done", "sm_exp_done",
         "sm_pempty_done", "sm_pfull_arrive"]
n = int((buf[0] > 0).sum())
t0 = buf[0][0]
print("tiles traced", n)
print("g   " + " ".join(f"{x:>16s}" for x in names) + "   | warp6: s_full ldtm exp pfull")
for g in range(min(n, 60)):
    row = [buf[i][g] - t0 if buf[i][g] else -1 for i in range(9)]
    row6 = [buf[i][g] - t0 if buf[i][g] else -1 for i in (10, 11, 12, 14)]
    print(f"{g:3d} " + " ".join(f"{x:16d}" for x in row) + "   | " + " ".join(f"{x:8d}" for x in row6))
d = np.diff(buf[8][:n])
print("median period (pfull arrive, warp2):", np.median(d[5:]))
names += ["-", "w6a", "w6b", "w6c", "w6d", "w6e", "mma_loop_top", "mma_k_full", "mma_s_empty", "pv_v_full"]
for a, b in [(15, 16), (16, 17), (17, 0), (1, 18), (18, 2), (2, 15), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8), (0, 4), (8, 1), (1, 2)]:
    x = buf[b][5:n - 5] - buf[a][5:n - 5] if not (a == 2 and b == 15) else buf[15][6:n - 4] - buf[2][5:n - 5]
    print(f"{names[a]:>16s} -> {names[b]:<16s} median {np.median(x):8.0f}")
