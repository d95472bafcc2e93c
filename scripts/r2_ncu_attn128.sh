mkdir -p gpurun_out
python scripts/attn_one.py vit fwd > gpurun_out/ncu_plain_vit.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/r02_attn_fwd_vit \
  python scripts/attn_one.py vit fwd > gpurun_out/ncu_vit.log 2>&1; echo "vit $?"
python scripts/attn_one.py cfg5_teacher fwd > gpurun_out/ncu_plain_c5.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/r02_attn_fwd_c5 \
  python scripts/attn_one.py cfg5_teacher fwd > gpurun_out/ncu_c5.log 2>&1; echo "c5 $?"
