# ncu evidence for the KD bench at the benched config (batch 64/rank): launch list, per-kernel
# rooflines, and an ncu --set full capture of the dominant GEMM shape (teacher gate/up + SwiGLU).
mkdir -p gpurun_out
O=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $O/ncu_plain_bench.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv -s 2800 -c 2600 \
  --log-file $O/r02_launches.csv $CMD > $O/ncu_ll.log 2>&1; echo "launch list $?"
$CMD > $O/ncu_plain_bench2.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed \
  --cache-control all --clock-control none --csv -s 2800 -c 2600 --log-file $O/r02_roof.csv $CMD > $O/ncu_roof.log 2>&1; echo "rooflines $?"
python scripts/gemm_prof.py 32768 11264 2048 swiglu_only > $O/ncu_plain_gemm.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm2_kernel -s 2 -c 1 -o $O/r02_gemm_gu \
  python scripts/gemm_prof.py 32768 11264 2048 swiglu_only > $O/ncu_gemm.log 2>&1; echo "gemm full $?"
python scripts/attn_one.py kd_teacher fwd > $O/ncu_plain_attn.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 2 -c 1 -o $O/r02_attn_fwd_kd \
  python scripts/attn_one.py kd_teacher fwd > $O/ncu_attn.log 2>&1; echo "attn full $?"
ls -la $O/r02_*
