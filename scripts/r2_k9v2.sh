#!/bin/bash
# K9 v2 (shared-memory-resident rows): parity, A/B against the streaming kernel, ncu traffic
set -x
python -m pytest tests/test_section_compute.py -m gpu -x -q -k kd_loss > gpurun_out/k9v2_test.log 2>&1
python scripts/kd_loss_bench.py > gpurun_out/k9v2_bench.jsonl 2>&1
MAESTRO_KD_IMPL=stream python scripts/kd_loss_bench.py > gpurun_out/k9v2_bench_stream.jsonl 2>&1
timeout 300 ncu --set full --clock-control none -k regex:kd_loss_smem -s 3 -c 1 -o gpurun_out/k9v2 -f python scripts/kd_loss_bench.py > gpurun_out/k9v2_ncu.log 2>&1
echo done
