"""K9 fused KL at the step's size (student micro-batch of 8 x 2048 tokens, 32k vocab): time and
achieved HBM GB/s (read t + s, write ds) against the measured copy bandwidth."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import kernels as K  # noqa: E402

T, V = 16384, 32000
t = (torch.randn(T, V, device="cuda") * 2).bfloat16()
s = (torch.randn(T, V, device="cuda") * 2).bfloat16()
loss = torch.empty(T, device="cuda")
for _ in range(3):
    ds = s.clone()
    K.kd_loss(t, ds, ds, loss, 1.0 / T)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ds = s.clone()
e0.record()
for _ in range(10):
    K.kd_loss(t, ds, ds, loss, 1.0 / T)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nbytes = 3 * T * V * 2
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(json.dumps({"T": T, "V": V, "ms": ms, "GBps": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / peak}))
