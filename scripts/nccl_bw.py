"""NCCL all-reduce bus bandwidth on this box (torchrun, one process per GPU): fp32 buffers of the
per-section gradient sizes, alone on the default stream and on a side stream next to a running
tcgen05 GEMM (the C2 situation).  Prints one JSON line from rank 0."""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = dist.get_world_size()
    out = {"world": n, "alone": {}, "beside_gemm": {}}
    for mb in (64, 551, 2048):
        x = torch.ones(mb * (1 << 20) // 4, device="cuda")
        for _ in range(3):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dist.all_reduce(x)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 5 / 1e3
        out["alone"][f"{mb}MB"] = 2 * (n - 1) / n * x.numel() * 4 / t / 1e9
    from paper_2605_10501_b200 import dense

    a = torch.randn(32768, 2048, device="cuda").bfloat16()
    w = torch.randn(11264, 2048, device="cuda").bfloat16()
    x = torch.ones(551 * (1 << 20) // 4, device="cuda")
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        dense.linear_fwd(a, w)
    with torch.cuda.stream(side):
        e0.record(side)
        dist.all_reduce(x)
        e1.record(side)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    out["beside_gemm"]["551MB"] = 2 * (n - 1) / n * x.numel() * 4 / t / 1e9
    if dist.get_rank() == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
