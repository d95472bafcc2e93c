#!/bin/bash
for c in teacher student both; do
  echo "== dec $c" >> gpurun_out/b3.log
  MAESTRO_ATTN_FWD=dec timeout 60 python scripts/diag_dec.py $c >> gpurun_out/b3.log 2>&1; echo "rc=$?" >> gpurun_out/b3.log
done
echo "== pp both" >> gpurun_out/b3.log
MAESTRO_ATTN_FWD=pp timeout 60 python scripts/diag_dec.py both >> gpurun_out/b3.log 2>&1; echo "rc=$?" >> gpurun_out/b3.log
echo done
