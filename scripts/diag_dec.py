"""Diagnose a stall of an attention forward variant at the cfg 2 step shapes:
python scripts/diag_dec.py <case>  (case: teacher | student | both | teacher_bwd)."""
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import attention as A  # noqa: E402


def make(nseq, L, H, Hk, dh=64):
    T = nseq * L
    cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
    q = torch.randn(T, H, dh, device="cuda").bfloat16()
    k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    o = torch.empty_like(q)
    return cu, q, k, v, o, A.plan(cu, T), L


def run(x, reps):
    cu, q, k, v, o, plan, L = x
    for _ in range(reps):
        A.attn_fwd(q, k, v, cu, L, True, o, 1 / math.sqrt(q.shape[2]), plan=plan)


case = sys.argv[1]
tshape = make(16, 2048, 32, 4)
sshape = make(8, 2048, 12, 12)
torch.cuda.synchronize()
t0 = time.time()
if case == "teacher":
    for i in range(5):
        run(tshape, 1)
        torch.cuda.synchronize()
        print("teacher", i, round(time.time() - t0, 2), flush=True)
elif case == "student":
    for i in range(5):
        run(sshape, 1)
        torch.cuda.synchronize()
        print("student", i, round(time.time() - t0, 2), flush=True)
else:
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for i in range(5):
        with torch.cuda.stream(s1):
            run(tshape, 2)
        with torch.cuda.stream(s2):
            run(sshape, 3)
        torch.cuda.synchronize()
        print("both", i, round(time.time() - t0, 2), flush=True)
print("ok", flush=True)
