#!/bin/bash
# forward exponential split (FWD_EMU_BITS: pairs of every 8 on the FMA pipe): A/B, interleaved reps
R=$(pwd)
for rep in 1 2; do
for v in base attn_emu_0x22 attn_emu_0x00 attn_emu_0xAA; do
  L=""
  [ "$v" != base ] && L=$R/paper_2605_10501_b200/_lib/$v/libmaestro_b200.so
  echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/a11_quick.jsonl
  (cd scripts && MAESTRO_LIB_PATH=$L timeout 300 python attn_quick.py >> $R/gpurun_out/a11_quick.jsonl 2>&1)
done
done
echo done
