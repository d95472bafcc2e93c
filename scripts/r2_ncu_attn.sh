mkdir -p gpurun_out
python scripts/attn_one.py kd_teacher fwd > gpurun_out/ncu_attn_plain.log 2>&1 && \
python scripts/attn_one.py vit fwd >> gpurun_out/ncu_attn_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/ncu_attn_kd_fwd python scripts/attn_one.py kd_teacher fwd > gpurun_out/ncu_attn1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/ncu_attn_vit_fwd python scripts/attn_one.py vit fwd > gpurun_out/ncu_attn2.log 2>&1 ; \
tail -3 gpurun_out/ncu_attn1.log gpurun_out/ncu_attn2.log
