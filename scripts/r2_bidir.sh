#!/bin/bash
R=$(pwd)
for rep in 1 2; do
  for v in dec pp base; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/bidir.jsonl
    (cd scripts && MAESTRO_ATTN_FWD=$v timeout 300 python attn_bidir64.py >> $R/gpurun_out/bidir.jsonl 2>&1)
  done
done
echo done
