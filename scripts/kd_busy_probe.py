"""Debug probe: GPU kernel-busy fraction of the single-GPU KD step (torch.profiler / CUPTI): union
of kernel intervals vs the step span, plus the longest idle gaps (where the device waits)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_10501_b200.executor import KDExecutor, synthetic_ids  # noqa: E402

ex = KDExecutor(n_gpus=1, batch_per_rank=64, seq=bench.SEQ, mbs=8, teacher_mbs=16)
ids = torch.from_numpy(synthetic_ids(ex.batch, bench.SEQ, 32000)).cuda()
for _ in range(2):
    ex.step(ids, want_loss=False)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ex.step(ids, want_loss=True)
    torch.cuda.synchronize()
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA")
busy, gaps, cur_s, cur_e, last = 0, [], None, None, ""
for s, e, n in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, last[:50], n[:50]))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    last = n
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
gaps.sort(reverse=True)
print({"span_ms": span / 1e3, "busy_ms": busy / 1e3, "busy_frac": busy / span, "kernels": len(iv),
       "idle_ms": (span - busy) / 1e3, "gaps_over_20us": sum(1 for g in gaps if g[0] > 20)})
for g in gaps[:12]:
    print(f"  gap {g[0]:8.1f} us after {g[1]!r} before {g[2]!r}")
