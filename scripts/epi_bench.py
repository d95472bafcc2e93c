"""Fused-epilogue GEMMs vs the plain bf16 epilogue on the step shapes (CUDA-event timed)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import dense  # noqa: E402
from paper_2605_10501_b200 import kernels as Kn  # noqa: E402
from paper_2605_10501_b200.transformer import rope_table  # noqa: E402


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


out = []
for M, N, K, kind in [(8192, 11264, 2048, "swiglu"), (8192, 2560, 2048, "rope"), (8192, 2048, 2048, "residual"),
                      (8192, 2048, 5632, "residual"), (8192, 6144, 768, "swiglu"), (8192, 2304, 768, "rope"),
                      (8192, 768, 768, "residual"), (8192, 768, 3072, "residual")]:
    a = torch.randn(M, K, device="cuda").bfloat16()  # normed activations ~ N(0, 1)
    w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()  # the model's N(0, 0.02) init
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    t_plain = timeit(lambda: dense.linear_fwd(a, w, c))
    if kind == "swiglu":
        s = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        t_f = timeit(lambda: dense.linear_fwd_swiglu(a, w, s, c))
        t_u = timeit(lambda: (dense.linear_fwd(a, w, c), Kn.swiglu(c, s)))
        t_ns = timeit(lambda: dense.linear_fwd_swiglu(a, w, s, store_gu=False))
    elif kind == "rope":
        pos = torch.arange(M, device="cuda", dtype=torch.int32) % 2048
        cs = rope_table(2048, 64, 10000.0, "cuda")
        t_f = timeit(lambda: dense.linear_fwd_rope(a, w, pos, cs, N - 512, c))
        t_u = timeit(lambda: (dense.linear_fwd(a, w, c), Kn.rope(c[:, : N - 512], pos, cs, (N - 512) // 64, 64)))
    else:
        r = torch.randn(M, N, device="cuda").bfloat16()
        t_f = timeit(lambda: dense.linear_fwd_residual(a, w, r, c))
        t_u = t_plain
    rec = {"shape": [M, N, K], "epilogue": kind, "plain_tflops": fl / t_plain / 1e12, "fused_tflops": fl / t_f / 1e12,
           "unfused_tflops": fl / t_u / 1e12}
    if kind == "swiglu":
        rec["fused_no_gu_store_tflops"] = fl / t_ns / 1e12
    print(json.dumps(rec), flush=True)
    out.append(rec)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/epi_bench.json").write_text(json.dumps(out, indent=1))
