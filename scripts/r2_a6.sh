#!/bin/bash
# ping-pong forward: parity (guarded), then A/B against base and dec
R=$(pwd)
MAESTRO_ATTN_FWD=pp timeout 240 python -m pytest tests/test_attention.py -m gpu -q -x > gpurun_out/a6_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a6_tests.log
if grep -q "tests rc=0" gpurun_out/a6_tests.log; then
  for rep in 1 2; do
    for v in base dec pp; do
      echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/a6_quick.jsonl
      (cd scripts && MAESTRO_ATTN_FWD=$v timeout 300 python attn_quick.py >> $R/gpurun_out/a6_quick.jsonl 2>&1)
    done
  done
fi
echo done
