#!/bin/bash
# K8 barrier addresses (u32 vs generic) A/B + K9 instruction trims; parity first
R=$(pwd)
ALT=$R/paper_2605_10501_b200/_lib/attn_bar_generic/libmaestro_b200.so
timeout 400 python -m pytest tests/test_attention.py tests/test_kd_loss_impls.py tests/test_section_compute.py -m gpu -q -x > gpurun_out/a4_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a4_tests.log
for rep in 1 2; do
  echo "{\"variant\": \"bar_u32\", \"rep\": $rep}" >> gpurun_out/a4_quick.jsonl
  (cd scripts && timeout 300 python attn_quick.py >> $R/gpurun_out/a4_quick.jsonl 2>&1)
  echo "{\"variant\": \"bar_generic\", \"rep\": $rep}" >> gpurun_out/a4_quick.jsonl
  (cd scripts && MAESTRO_LIB_PATH=$ALT timeout 300 python attn_quick.py >> $R/gpurun_out/a4_quick.jsonl 2>&1)
done
timeout 120 python scripts/kd_loss_bench.py > gpurun_out/a4_k9.jsonl 2>&1
MAESTRO_KD_IMPL=stream timeout 120 python scripts/kd_loss_bench.py >> gpurun_out/a4_k9.jsonl 2>&1
echo done
