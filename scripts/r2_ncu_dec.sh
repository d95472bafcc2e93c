#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/a13_dec -f python scripts/attn_one.py kd_teacher fwd > gpurun_out/a13_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:kd_loss_smem -s 3 -c 1 -o gpurun_out/a13_k9 -f python scripts/kd_loss_bench.py > gpurun_out/a13_ncu2.log 2>&1
echo done
