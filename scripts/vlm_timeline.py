import os, sys, json
sys.path.insert(0, "/root/repo")
import torch, torch.distributed as dist
from paper_2605_10501_b200.vlm import VLMGroupExecutor, vlm_host_batch
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ex = VLMGroupExecutor(dist.get_world_size(), batch_per_llm_rank=64)
hb = vlm_host_batch(ex.batch, seed=0)
for _ in range(3): st = ex.step(hb)
tl = ex.timeline()
out = [None] * dist.get_world_size()
dist.all_gather_object(out, (ex.role, st.step_ms, tl))
if dist.get_rank() == 0:
    for role, ms, tl in out:
        print(role, round(ms, 2), [(n, round(a, 2), round(b, 2)) for n, a, b in tl])
dist.destroy_process_group()
