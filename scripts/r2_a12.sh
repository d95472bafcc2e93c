#!/bin/bash
# four 32-column decoupled groups (dec4): parity vs shared tile (subprocess, guarded), then A/B
R=$(pwd)
MAESTRO_ATTN_FWD=dec4 timeout 300 python -m pytest tests/test_attention.py -m gpu -q -x -k "not hd128" > gpurun_out/a12_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a12_tests.log
timeout 600 python -m pytest tests/test_attention_variants.py -m gpu -q -x -k dec4 >> gpurun_out/a12_tests.log 2>&1
echo "variants rc=$?" >> gpurun_out/a12_tests.log
if grep -q "tests rc=0" gpurun_out/a12_tests.log; then
  for rep in 1 2; do
    for v in dec dec4; do
      echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/a12_quick.jsonl
      (cd scripts && MAESTRO_ATTN_FWD=$v timeout 300 python attn_quick.py >> $R/gpurun_out/a12_quick.jsonl 2>&1)
    done
  done
fi
echo done
