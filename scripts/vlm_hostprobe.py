"""Debug probe: host time spent in the VLM group executor's handoff / upload calls (calls > 0.3 ms)."""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import mq, vlm  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
LOG = []
T0 = [0.0]


def wrap(obj, name, label):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        dt = (time.perf_counter() - t) * 1e3
        if dt > 0.3:
            LOG.append((label, round((t - T0[0]) * 1e3, 2), round(dt, 2)))
        return r

    setattr(obj, name, g)


wrap(mq.Endpoint, "pull", "pull")
wrap(mq.Channel, "push", "push")
wrap(vlm, "_h2d", "h2d")
ex = vlm.VLMGroupExecutor(dist.get_world_size(), batch_per_llm_rank=64)
hb = vlm.vlm_host_batch(ex.batch, seed=0)
for _ in range(3):
    LOG.clear()
    T0[0] = time.perf_counter()
    st = ex.step(hb)
    host_ms = (time.perf_counter() - T0[0]) * 1e3
out = [None] * dist.get_world_size()
dist.all_gather_object(out, (ex.role, round(st.step_ms, 2), round(host_ms, 2), LOG[:40]))
if dist.get_rank() == 0:
    for o in out:
        print(o)
dist.destroy_process_group()
