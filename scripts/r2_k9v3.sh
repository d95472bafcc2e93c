#!/bin/bash
# K9 v3 (3 CTAs/SM, cluster row slices) + K3 fast path: parity, timing, ncu
timeout 300 python -m pytest tests/test_section_compute.py -m gpu -x -q -k kd_loss > gpurun_out/k9v3_test.log 2>&1
timeout 120 python scripts/kd_loss_bench.py > gpurun_out/k9v3_bench.jsonl 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "sched or plan or wavefront or golden or device" > gpurun_out/k3_test.log 2>&1
timeout 200 python scripts/plan_bench.py > gpurun_out/k3_plan_bench.jsonl 2>&1
timeout 300 ncu --set full --clock-control none -k regex:kd_loss_smem -s 3 -c 1 -o gpurun_out/k9v3 -f python scripts/kd_loss_bench.py > gpurun_out/k9v3_ncu.log 2>&1
echo done
