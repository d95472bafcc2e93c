#!/bin/bash
# A/B: warp-level vs per-thread barrier arrives in K8 (same box, interleaved), peer test, ncu of fwd
R=$(pwd)
ALT=$R/paper_2605_10501_b200/_lib/attn_thread_arrive/libmaestro_b200.so
for rep in 1 2; do
  echo "{\"variant\": \"warp_arrive\", \"rep\": $rep}" >> gpurun_out/a2_quick.jsonl
  (cd scripts && timeout 300 python attn_quick.py >> $R/gpurun_out/a2_quick.jsonl 2>&1)
  echo "{\"variant\": \"thread_arrive\", \"rep\": $rep}" >> gpurun_out/a2_quick.jsonl
  (cd scripts && MAESTRO_LIB_PATH=$ALT timeout 300 python attn_quick.py >> $R/gpurun_out/a2_quick.jsonl 2>&1)
done
timeout 200 python scripts/peer_same_gpu.py > gpurun_out/peer_same_gpu.log 2>&1
timeout 300 python -m pytest tests/test_mq.py -m gpu -q -x -k two_processes > gpurun_out/a2_mq.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/a2_attn_fwd -f python scripts/attn_one.py > gpurun_out/a2_ncu.log 2>&1
echo done
