#!/bin/bash
for rep in 1 2; do
  for v in 1 0; do
    echo "{\"pdl\": $v, \"rep\": $rep}" >> gpurun_out/pdl4.jsonl
    MAESTRO_PDL=$v timeout 900 python bench.py --workload section --graph vlm7b --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/pdl4.jsonl
    MAESTRO_PDL=$v timeout 900 python bench.py --workload section --graph omni --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/pdl4.jsonl
  done
done
echo done
