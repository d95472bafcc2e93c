#!/bin/bash
# bisect the cfg 2 bench stall: default / streaming K9 / shared-tile attention forward
for v in "default" "MAESTRO_KD_IMPL=stream" "MAESTRO_ATTN_FWD=base" "MAESTRO_KD_IMPL=stream MAESTRO_ATTN_FWD=base"; do
  echo "== $v" >> gpurun_out/b2.log
  start=$(date +%s)
  env $([ "$v" != default ] && echo $v) timeout 240 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b2_out.json 2>> gpurun_out/b2.log
  echo "rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/b2.log
  tail -c 300 gpurun_out/b2_out.json >> gpurun_out/b2.log; echo >> gpurun_out/b2.log
done
echo done
