#!/bin/bash
# decoupled-column-group forward: parity (guarded), then A/B vs the shared-tile forward
R=$(pwd)
MAESTRO_ATTN_FWD=dec timeout 300 python -m pytest tests/test_attention.py -m gpu -q -x > gpurun_out/a5_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a5_tests.log
if grep -q "tests rc=0" gpurun_out/a5_tests.log; then
  for rep in 1 2; do
    for v in base dec; do
      echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/a5_quick.jsonl
      (cd scripts && MAESTRO_ATTN_FWD=$v timeout 300 python attn_quick.py >> $R/gpurun_out/a5_quick.jsonl 2>&1)
    done
  done
  for ns in 0 1000; do
    echo "{\"variant\": \"dec_stagger$ns\", \"rep\": 1}" >> gpurun_out/a5_quick.jsonl
    (cd scripts && MAESTRO_ATTN_FWD=dec MAESTRO_ATTN_DEC_STAGGER_NS=$ns timeout 300 python attn_quick.py >> $R/gpurun_out/a5_quick.jsonl 2>&1)
  done
fi
echo done
