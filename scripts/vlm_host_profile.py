"""Debug probe: host-side cProfile of the single-GPU VLM step (which Python calls cost the most)."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200.vlm import VLMExecutor, vlm_host_batch  # noqa: E402

ex = VLMExecutor(batch=64, mbs_llm=32, mbs_vit=32)
hb = vlm_host_batch(64, seed=0)
for _ in range(3):
    ex.step(hb, want_loss=False, next_hb=hb)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    ex.step(hb, want_loss=False, next_hb=hb)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
