"""VLM on 2 GPUs, disjoint section groups or both sections data-parallel per GPU: same losses as
the co-resident single-GPU step.

Runs scripts/vlm_dist_check.py under torchrun when the box has >= 2 GPUs (skipped otherwise).
Tolerance: the two layouts run the same kernels on the same micro-batches; only the fp32
reduction order of the cross-rank loss / gradient sums differs -> 1e-3 relative on the loss.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("layout", ["disjoint", "colocated"])
def test_vlm_layouts_match_single_gpu(layout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(ROOT / "scripts" / "vlm_dist_check.py")]
    if layout == "colocated":
        cmd.append("--colocated")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    assert out.returncode == 0, out.stderr[-3000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)
    assert res["max_rel_diff"] < 1e-3, res
