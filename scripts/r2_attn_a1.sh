#!/bin/bash
# attention: warp-level barrier arrives + group stagger knob -- parity + quick TFLOP/s
R=$(pwd)
timeout 400 python -m pytest tests/test_attention.py -m gpu -q -x > gpurun_out/a1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a1_tests.log
for ns in 0 300 700; do
  echo "{\"stagger_ns\": $ns}" >> gpurun_out/a1_quick.jsonl
  (cd scripts && MAESTRO_ATTN_STAGGER_NS=$ns timeout 300 python attn_quick.py >> $R/gpurun_out/a1_quick.jsonl 2>&1)
done
echo done
timeout 200 python scripts/peer_same_gpu.py > gpurun_out/peer_same_gpu.log 2>&1
