"""Microbenchmark: tcgen05 GEMM (K7) vs cuBLAS (torch.matmul) on training shapes."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import dense  # noqa: E402


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


def main():
    shapes = [(8192, 8192, 8192)]
    if "--student" in sys.argv:  # the student's per-micro-batch GEMMs (T = mbs x 2048; mbs 8 by default)
        T = 2048 * int(sys.argv[sys.argv.index("--student") + 1]) if len(sys.argv) > sys.argv.index("--student") + 1 else 16384
        shapes = [(T, 2304, 768), (T, 768, 768), (T, 6144, 768), (T, 768, 3072), (T, 32000, 768)]
    elif "--step" in sys.argv:  # the exact per-micro-batch GEMMs of the KD step (T = 4 x 2048)
        shapes += [(8192, 2560, 2048), (8192, 2048, 2048), (8192, 11264, 2048), (8192, 2048, 5632),
                   (8192, 32000, 2048), (8192, 2304, 768), (8192, 768, 768), (8192, 6144, 768),
                   (8192, 768, 3072), (8192, 32000, 768)]
    else:
        shapes += [(16384, 2048, 2048), (16384, 5632, 2048), (16384, 2048, 5632), (16384, 768, 768),
                   (16384, 3072, 768), (16384, 32000, 2048), (16384, 32000, 768)]
    out = []
    for M, N, K in shapes:
        a = torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(N, K, device="cuda").bfloat16()
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        t_ours = timeit(lambda: dense.linear_fwd(a, b, c))
        t_cub = timeit(lambda: torch.matmul(a, b.t(), out=c))
        dy = torch.randn(M, N, device="cuda").bfloat16()
        dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
        bt = b.t().contiguous()  # the training path keeps a K-major (transposed) weight copy
        t_dg = timeit(lambda: dense.linear_dgrad(dy, b, dx, wt=bt))
        dw = torch.zeros(N, K, device="cuda")
        t_wg = timeit(lambda: dense.linear_wgrad(dy, a, dw))
        t_cub_wg = timeit(lambda: torch.matmul(dy.t(), a))
        rec = {"shape": [M, N, K], "fwd_tflops": fl / t_ours / 1e12, "cublas_tflops": fl / t_cub / 1e12,
               "dgrad_tflops": fl / t_dg / 1e12, "wgrad_tflops": fl / t_wg / 1e12,
               "cublas_wgrad_tflops": fl / t_cub_wg / 1e12}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/gemm_bench.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
