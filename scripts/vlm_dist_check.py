"""Layout equivalence of the VLM step ("identical model updates regardless of
reorder"): the disjoint-group executor at N GPUs vs the co-resident executor on one GPU, same
batch and seeds.  Run under torchrun; rank 0 prints one JSON line.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/vlm_dist_check.py
    ... scripts/vlm_dist_check.py --colocated   (both sections DP on every GPU, same batch per rank:
                                                 the averaged gradients equal the single-GPU ones)
"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200.vlm import VLMExecutor, VLMGroupExecutor, vlm_host_batch  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
world, rank = dist.get_world_size(), dist.get_rank()
steps = 3
if "--colocated" in sys.argv:
    ex = VLMExecutor(batch=64, mbs_llm=8, mbs_vit=8, lr=1e-3, dp_group=dist.group.WORLD)
else:
    ex = VLMGroupExecutor(world, batch_per_llm_rank=64 // max(1, {2: 1, 4: 3, 8: 6}[world]) if world > 2 else 64,
                          mbs_llm=8, mbs_vit=8, lr=1e-3)
hb = vlm_host_batch(ex.batch, seed=0)
group = [ex.step(hb).loss for _ in range(steps)]
dist.barrier()
if rank == 0:
    single = VLMExecutor(batch=ex.batch, mbs_llm=8, mbs_vit=ex.mbs_vit, lr=1e-3)
    ref = [single.step(hb).loss for _ in range(steps)]
    rel = max(abs(a - b) / abs(b) for a, b in zip(group, ref))
    print(json.dumps({"world": world, "batch": ex.batch, "group_losses": group, "single_gpu_losses": ref,
                      "max_rel_diff": rel}), flush=True)
dist.barrier()
dist.destroy_process_group()
