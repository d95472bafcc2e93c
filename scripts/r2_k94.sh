#!/bin/bash
R=$(pwd)
L=$R/paper_2605_10501_b200/_lib/k9_4cta/libmaestro_b200.so
MAESTRO_LIB_PATH=$L MAESTRO_KD_IMPL=smem timeout 300 python -m pytest tests/test_section_compute.py -m gpu -q -x -k kd_loss > gpurun_out/k94_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k94_tests.log
for rep in 1 2; do
  echo "{\"variant\": \"base\", \"rep\": $rep}" >> gpurun_out/k94.jsonl
  timeout 120 python scripts/kd_loss_bench.py >> gpurun_out/k94.jsonl 2>&1
  echo "{\"variant\": \"4cta_192\", \"rep\": $rep}" >> gpurun_out/k94.jsonl
  MAESTRO_LIB_PATH=$L MAESTRO_KD_IMPL=smem timeout 120 python scripts/kd_loss_bench.py >> gpurun_out/k94.jsonl 2>&1
done
echo done
