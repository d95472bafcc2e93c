"""K9 implementations selected by MAESTRO_KD_IMPL (read once per process, so each runs in a
subprocess): the shared-memory-resident cluster kernel at every cluster size it supports and the
streaming kernel, both against the fp32 reference (max-normalised error: loss 1e-4, ds 1e-2 as in
test_section_compute)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from oracle import torch_ref as R
from paper_2605_10501_b200 import kernels as K
def rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6))
for T, V in ((17, 32000), (9, 40000), (5, 128256), (3, 4104)):
    torch.manual_seed(V)
    t = (3 * torch.randn(T, V, device="cuda")).bfloat16()
    s = (3 * torch.randn(T, V, device="cuda")).bfloat16()
    ss = s.float().clone().requires_grad_(True)
    ref = R.kd_loss(t.float(), ss)
    (ref.sum() * 0.5).backward()
    loss = torch.empty(T, device="cuda")
    ds = torch.empty_like(s)
    K.kd_loss(t, s, ds, loss, grad_scale=0.5)
    torch.cuda.synchronize()
    assert rel(loss, ref) < 1e-4, (T, V, rel(loss, ref))
    assert rel(ds, ss.grad) < 1e-2, (T, V, rel(ds, ss.grad))
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("impl", ["smem", "stream"])
def test_kd_loss_impl(impl):
    env = dict(os.environ, MAESTRO_KD_IMPL=impl)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
