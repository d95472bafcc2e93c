"""Step-by-step progress of the cfg 5 KD step and the hd128 attention at its shapes, with a
watchdog that dumps the stack if anything stalls."""
import faulthandler
import math
import os
import sys
import time
from pathlib import Path

faulthandler.dump_traceback_later(int(os.environ.get("DIAG_SECS", "240")), exit=True)
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402


def log(*a):
    print(f"[{time.time() - T0:7.2f}s]", *a, flush=True)


T0 = time.time()


def attn(L, nseq, H, Hk, dh, causal, bwd):
    from paper_2605_10501_b200 import attention as A

    T = L * nseq
    cu = torch.arange(0, T + 1, L, dtype=torch.int32, device="cuda")
    q = torch.randn(T, H, dh, device="cuda").bfloat16()
    k = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    v = torch.randn(T, Hk, dh, device="cuda").bfloat16()
    o = torch.empty_like(q)
    plan = A.plan(cu, T)
    lse = A.attn_fwd(q, k, v, cu, L, causal, o, 1 / math.sqrt(dh), plan=plan)
    torch.cuda.synchronize()
    log("attn fwd ok", L, nseq, H, Hk, dh, causal)
    if bwd:
        do = torch.randn_like(q)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        A.attn_bwd(do, q, k, v, o, lse, cu, L, causal, dq, dk, dv, 1 / math.sqrt(dh), plan=plan)
        torch.cuda.synchronize()
        log("attn bwd ok")


def main():
    which = sys.argv[1]
    if which == "attn":
        attn(8192, 2, 32, 8, 128, True, False)
        attn(8192, 1, 32, 8, 128, True, True)
        attn(4096, 2, 28, 4, 128, True, True)
        attn(4096, 4, 16, 16, 128, False, True)
        attn(8192, 1, 32, 8, 64, True, True)
    elif which == "kd8b":
        import dataclasses

        from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids
        from paper_2605_10501_b200.transformer import SHAPES

        nl = int(os.environ.get("LAYERS", "0"))
        if nl:
            SHAPES["t_dbg"] = dataclasses.replace(SHAPES["llama3_8b"], layers=nl)
            SHAPES["s_dbg"] = dataclasses.replace(SHAPES["llama32_1b"], layers=nl)
        ex = KDExecutor(n_gpus=1, batch_per_rank=2, seq=8192, mbs=1, teacher="t_dbg" if nl else "llama3_8b",
                        student="s_dbg" if nl else "llama32_1b", recipe="kd_8b", teacher_mbs=2)
        log("executor built", torch.cuda.memory_allocated() / 2**30, "GiB")
        ids = torch.from_numpy(synthetic_ids(2, 8192, 128256)).cuda()
        for i in range(2):
            st = ex.step(ids)
            log("step", i, st.loss, st.step_ms, "ms", torch.cuda.max_memory_allocated() / 2**30, "GiB peak")
    elif which == "vlm7b":
        from paper_2605_10501_b200 import graph_workloads as W

        ex = W.vlm7b_executor(layers=int(os.environ.get("LAYERS", "2")))
        log("executor built", torch.cuda.memory_allocated() / 2**30, "GiB")
        gb = W.vlm7b_batch(4, seed=0, vocab=W.QWEN_7B.vocab, patch_dim=W.PATCH_DIM)
        log("batch", gb.lens.tolist(), gb.up["vit"].in_len.tolist())
        for i in range(2):
            st = ex.step(gb)
            log("step", i, st.loss, st.step_ms, "ms", torch.cuda.max_memory_allocated() / 2**30, "GiB peak")


if __name__ == "__main__":
    main()
