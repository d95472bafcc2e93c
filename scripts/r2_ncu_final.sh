# ncu evidence for the final KD bench (batch 64/rank): launch list + per-kernel rooflines
mkdir -p gpurun_out
O=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $O/ncuf_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv -s 2800 -c 2600 \
  --log-file $O/r02_launches_v2.csv $CMD > $O/ncuf_ll.log 2>&1; echo "launch list $?"
$CMD > $O/ncuf_plain2.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed \
  --cache-control all --clock-control none --csv -s 2800 -c 2600 --log-file $O/r02_roof_v2.csv $CMD > $O/ncuf_roof.log 2>&1; echo "rooflines $?"
ls -la $O/r02_*v2*
