"""Diag-only: per-iteration pipeline timeline of attention-backward CTA 0 (lib built with the
backward trace hooks exporting maestro_diag_trace)."""
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
q, k, v = (torch.randn(T, h, dh, device="cuda").bfloat16() for h in (H, Hk, Hk))
o = torch.empty_like(q)
sc = 1 / math.sqrt(dh)
lse = A.attn_fwd(q, k, v, cu, L, True, o, sc)
do = torch.randn_like(q)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
for _ in range(3):
    A.attn_bwd(do, q, k, v, o, lse, cu, L, True, dq, dk, dv, sc)
torch.cuda.synchronize()
buf = np.zeros((20, 1024), dtype=np.int64)
assert _native.lib().maestro_diag_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["M:p_ready", "M:dV_iss", "M:S+1_iss", "M:ds_ready", "M:dq_empty", "M:dKdQ_iss", "M:dP+1_iss",  # order per build
         "s:s_full", "s:p_free", "s:P1_done", "s:dp_full", "s:ds_free", "s:P2_done", "d:dq_full", "d:done"]
n = int((buf[0] > 0).sum())
t0 = buf[0][0]
print("iterations traced", n)
print("gi  " + " ".join(f"{x:>11s}" for x in names))
for g in range(min(n, 40)):
    print(f"{g:3d} " + " ".join(f"{(buf[i][g] - t0) if buf[i][g] else -1:11d}" for i in range(15)))
d = np.diff(buf[12][:n])
print("median period (P2 done):", np.median(d[5:]))
order = [7, 8, 9, 10, 11, 12]
for a, b in zip(order, order[1:]):
    print(f"{names[a]:>12s} -> {names[b]:<12s} median {np.median(buf[b][5:n-5] - buf[a][5:n-5]):8.0f}")
for a, b in [(2, 0), (0, 1), (1, 3), (3, 4), (4, 5), (5, 6), (9, 0), (12, 3), (13, 14), (7, 2)]:
    print(f"{names[a]:>12s} -> {names[b]:<12s} median {np.median(buf[b][5:n-5] - buf[a][5:n-5]):8.0f}")
for a, b in [(4, 19), (19, 5), (18, 15), (15, 16), (16, 17)]:
    print(f"issue_s {a}->{b} median {np.median(buf[b][5:n-5] - buf[a][5:n-5]):8.0f}")
print("issue_s start -> s_full seen", np.median(buf[7][5:n-5] - buf[18][5:n-5]))
x = buf[0][6:n-4] - buf[6][5:n-5]
print(f"{'M:dP+1_iss':>12s} -> next p_ready median {np.median(x):8.0f}")
x = buf[7][6:n-4] - buf[12][5:n-5]
print(f"{'s:P2_done':>12s} -> next s_full median {np.median(x):8.0f}")
