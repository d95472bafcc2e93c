"""Capture the first head_dim-128 attention forward call of the cfg 5 KD step (1-layer teacher),
then replay it in fresh processes under variations to isolate a stall."""
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
DUMP = "/tmp/attn_dump.pt"


def capture():
    import dataclasses
    import faulthandler

    import torch

    faulthandler.dump_traceback_later(100, exit=True)
    from paper_2605_10501_b200 import attention as A
    from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids
    from paper_2605_10501_b200.transformer import SHAPES

    orig = A.attn_fwd

    def spy(q, k, v, cu, max_len, causal, out, scale, plan=None):
        if q.shape[-1] == 128 and not os.path.exists(DUMP):
            torch.cuda.synchronize()
            torch.save({"q": q.clone(), "k": k.clone(), "v": v.clone(), "cu": cu.clone(), "max_len": max_len,
                        "causal": causal, "scale": scale, "qs": q.stride(0), "ks": k.stride(0),
                        "qkv_base_off": (k.data_ptr() - q.data_ptr(), v.data_ptr() - q.data_ptr())}, DUMP)
            print("dumped", q.shape, k.shape, cu.tolist(), q.stride(), k.stride(), flush=True)
        return orig(q, k, v, cu, max_len, causal, out, scale, plan=plan)

    A.attn_fwd = spy
    SHAPES["t_dbg"] = dataclasses.replace(SHAPES["llama3_8b"], layers=1)
    SHAPES["s_dbg"] = dataclasses.replace(SHAPES["llama32_1b"], layers=1)
    ex = KDExecutor(n_gpus=1, batch_per_rank=2, seq=8192, mbs=1, teacher="t_dbg", student="s_dbg", recipe="kd_8b",
                    teacher_mbs=2)
    ids = torch.from_numpy(synthetic_ids(2, 8192, 128256)).cuda()
    ex.step(ids)
    print("capture step finished", flush=True)


def replay(variant):
    import math

    import torch

    from paper_2605_10501_b200 import attention as A

    d = torch.load(DUMP)
    q, k, v, cu = d["q"], d["k"], d["v"], d["cu"]
    T, H, dh = q.shape
    if variant == "contig":
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    if variant == "pitched":  # rebuild the fused-QKV pitch layout
        Hk = k.shape[1]
        buf = torch.empty(T, (H + 2 * Hk) * dh, device="cuda", dtype=torch.bfloat16)
        buf[:, : H * dh] = q.reshape(T, -1)
        buf[:, H * dh: (H + Hk) * dh] = k.reshape(T, -1)
        buf[:, (H + Hk) * dh:] = v.reshape(T, -1)
        q = buf[:, : H * dh].view(T, H, dh)
        k = buf[:, H * dh: (H + Hk) * dh].view(T, Hk, dh)
        v = buf[:, (H + Hk) * dh:].view(T, Hk, dh)
    if variant == "randn":
        q, k, v = torch.randn_like(q), torch.randn_like(k), torch.randn_like(v)
    if variant == "scaled":
        q = (q.float() * 8).bfloat16()
    o = torch.empty(T, H, dh, device="cuda", dtype=torch.bfloat16)
    plan = A.plan(cu, T)
    A.attn_fwd(q, k, v, cu, d["max_len"], d["causal"], o, d["scale"], plan=plan)
    torch.cuda.synchronize()
    s = (q[:2048, 0].float() @ k[:2048, 0].float().t()) * d["scale"] * 1.4427
    print(variant, "ok; |s| max", s.abs().max().item(), "o finite", torch.isfinite(o).all().item(), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "capture":
        capture()
    elif sys.argv[1] == "replay":
        replay(sys.argv[2])
    else:
        for var in ("asis", "contig", "pitched", "randn", "scaled"):
            t0 = time.time()
            r = subprocess.run([sys.executable, __file__, "replay", var], capture_output=True, text=True, timeout=None
                               if False else 90) if False else None
            try:
                r = subprocess.run([sys.executable, __file__, "replay", var], capture_output=True, text=True,
                                   timeout=60)
                print(var, "rc", r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-300:], flush=True)
            except subprocess.TimeoutExpired:
                print(var, "TIMEOUT after", time.time() - t0, flush=True)
