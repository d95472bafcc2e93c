#!/bin/bash
R=$(pwd)
timeout 300 python -m pytest tests/test_section_compute.py tests/test_kd_loss_impls.py -m gpu -q -x -k "kd_loss" > gpurun_out/k9s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k9s_tests.log
for rep in 1 2; do
  echo "{\"variant\": \"sleep\", \"rep\": $rep}" >> gpurun_out/k9s.jsonl
  timeout 120 python scripts/kd_loss_bench.py >> gpurun_out/k9s.jsonl 2>&1
  echo "{\"variant\": \"spin\", \"rep\": $rep}" >> gpurun_out/k9s.jsonl
  MAESTRO_LIB_PATH=$R/paper_2605_10501_b200/_lib/k9_spin/libmaestro_b200.so timeout 120 python scripts/kd_loss_bench.py >> gpurun_out/k9s.jsonl 2>&1
done
echo done
