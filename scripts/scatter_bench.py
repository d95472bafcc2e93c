"""K6 scatter / gather at cfg 3 sizes (Qwen2.5-VL-7B-shaped: 1024 merged tokens x 3584 per image):
achieved HBM GB/s (read + write bytes / CUDA-event time) against the measured copy bandwidth."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import kernels as K  # noqa: E402


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


peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
out = []
for n_img, tok, d in [(32, 1024, 3584), (64, 49, 768), (8, 1024, 3584)]:
    rows = n_img * tok
    T = rows * 3  # packed stream: images interleaved with text
    src = torch.randn(rows, d, device="cuda").bfloat16()
    dst = torch.zeros(T, d, device="cuda", dtype=torch.bfloat16)
    sr = torch.arange(rows, device="cuda", dtype=torch.int32)
    dr = (torch.randperm(T // tok, device="cuda")[:n_img].sort().values[:, None] * tok
          + torch.arange(tok, device="cuda")[None, :]).reshape(-1).to(torch.int32)
    t_f = timeit(lambda: K.scatter_rows(src, dst, sr, dr))
    assert torch.equal(dst[dr.long()], src)
    back = torch.empty_like(src)
    seg = torch.arange(rows + 1, device="cuda", dtype=torch.int32)
    t_b = timeit(lambda: K.gather_rows_bwd(dst, back, seg, dr))
    assert torch.equal(back, src)
    nbytes = 2 * rows * d * 2
    rec = {"images": n_img, "tokens_per_image": tok, "d": d, "bytes_per_call": nbytes,
           "scatter_GBps": nbytes / t_f / 1e9, "gather_bwd_GBps": nbytes / t_b / 1e9, "hbm_peak_GBps": peak,
           "scatter_frac": nbytes / t_f / 1e9 / peak, "gather_frac": nbytes / t_b / 1e9 / peak}
    print(json.dumps(rec), flush=True)
    out.append(rec)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/scatter_bench.json").write_text(json.dumps(out, indent=1))
