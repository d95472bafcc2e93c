#!/bin/bash
# KD micro-batch sizes: (student mbs, teacher mbs) A/B on one box, interleaved
for rep in 1 2; do
for cfg in "8 16" "16 16" "16 32" "8 32"; do
  set -- $cfg
  echo "{\"mbs\": $1, \"tmbs\": $2, \"rep\": $rep}" >> gpurun_out/mbs.jsonl
  timeout 400 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --mbs $1 --teacher-mbs $2 2>/dev/null | tail -1 | cut -c1-400 >> gpurun_out/mbs.jsonl
done
done
echo done
