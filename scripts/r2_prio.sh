#!/bin/bash
for rep in 1 2; do
  for v in none teacher; do
    echo "{\"prio\": \"$v\", \"rep\": $rep}" >> gpurun_out/prio2.jsonl
    MAESTRO_STREAM_PRIORITY=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/prio2.jsonl
    MAESTRO_STREAM_PRIORITY=$v timeout 600 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/prio2.jsonl
  done
done
echo done
