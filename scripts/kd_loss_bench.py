"""K9 (fused KL) at the cfg 2 and cfg 5 shapes: GB/s on algorithmic bytes (read t, s; write ds)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import kernels as K  # noqa: E402


def main():
    for T, V in ((16384, 32000), (8192, 128256)):
        t = torch.randn(T, V, device="cuda").bfloat16()
        s = torch.randn(T, V, device="cuda").bfloat16()
        loss = torch.empty(T, device="cuda")
        for _ in range(3):
            K.kd_loss(t, s, s, loss, 1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            K.kd_loss(t, s, s, loss, 1.0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"T": T, "V": V, "ms": ms, "GBps": 3 * T * V * 2 / (ms / 1e3) / 1e9}), flush=True)
        del t, s


if __name__ == "__main__":
    main()
