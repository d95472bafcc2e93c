#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pdl5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl5_tests.log
if grep -q "rc=0" gpurun_out/pdl5_tests.log; then
for rep in 1 2; do
  for v in 1 0; do
    echo "{\"pdl\": $v, \"rep\": $rep}" >> gpurun_out/pdl5.jsonl
    MAESTRO_PDL=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/pdl5.jsonl
    MAESTRO_PDL=$v timeout 900 python bench.py --workload section --graph vlm7b --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/pdl5.jsonl
  done
done
fi
echo done
