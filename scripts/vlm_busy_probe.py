"""Debug probe: GPU kernel-busy fraction of the single-GPU VLM step (torch.profiler / CUPTI):
union of kernel intervals vs the step's wall span -> is the step host-bound?"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200.vlm import VLMExecutor, vlm_host_batch  # noqa: E402

ex = VLMExecutor(batch=64, mbs_llm=32, mbs_vit=32)
hb = vlm_host_batch(64, seed=0)
for _ in range(3):
    ex.step(hb, want_loss=False, next_hb=hb)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    for _ in range(5):
        ex.step(hb, want_loss=False, next_hb=hb)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
iv = sorted((e.time_range.start, e.time_range.end) for e in prof.events() if e.device_type.name == "CUDA")
busy, cur_s, cur_e = 0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print({"steps": 5, "wall_ms_per_step": wall * 1e3 / 5, "gpu_span_ms_per_step": span / 1e3 / 5,
       "gpu_busy_ms_per_step": busy / 1e3 / 5, "busy_frac_of_span": busy / max(span, 1), "kernels": len(iv)})
