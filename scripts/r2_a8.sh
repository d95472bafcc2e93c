#!/bin/bash
# mbarrier try_wait suspend-time hint in the attention kernels: A/B on one box
R=$(pwd)
for v in base attn_susp_1ms attn_susp_20us; do
  L=""
  [ "$v" != base ] && L=$R/paper_2605_10501_b200/_lib/$v/libmaestro_b200.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/a8_quick.jsonl
  (cd scripts && MAESTRO_LIB_PATH=$L timeout 300 python attn_quick.py >> $R/gpurun_out/a8_quick.jsonl 2>&1)
done
MAESTRO_LIB_PATH=$R/paper_2605_10501_b200/_lib/attn_susp_1ms/libmaestro_b200.so timeout 300 python -m pytest tests/test_attention.py -m gpu -q -x > gpurun_out/a8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/a8_tests.log

for v in base gemm_susp_1ms; do
  L=""
  [ "$v" != base ] && L=$R/paper_2605_10501_b200/_lib/$v/libmaestro_b200.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/a8_gemm.jsonl
  MAESTRO_LIB_PATH=$L timeout 300 python scripts/gemm_bench.py --student 8 >> gpurun_out/a8_gemm.jsonl 2>&1
  MAESTRO_LIB_PATH=$L timeout 300 python scripts/gemm_bench.py >> gpurun_out/a8_gemm.jsonl 2>&1
done
echo done
