#!/bin/bash
# forward producer (TMA/MMA warp) sleep-waits: A/B, two reps interleaved
R=$(pwd)
for rep in 1 2; do
for v in base attn_prod_sleep; do
  L=""
  [ "$v" != base ] && L=$R/paper_2605_10501_b200/_lib/$v/libmaestro_b200.so
  echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/a10_quick.jsonl
  (cd scripts && MAESTRO_LIB_PATH=$L timeout 300 python attn_quick.py >> $R/gpurun_out/a10_quick.jsonl 2>&1)
done
done
echo done
