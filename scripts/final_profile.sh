# Round-end measurement pass on one GPU: GPU tests, bench lines (KD default + VLM), KD launch
# list, KD per-kernel rooflines, ncu --set full of attention fwd/bwd and the teacher gate/up GEMM.
set -u
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/final_tests.log 2>&1; tail -1 $O/final_tests.log
timeout 600 python bench.py > $O/final_bench_kd.json 2> $O/final_bench_kd.err
timeout 600 python bench.py --workload vlm > $O/final_bench_vlm.json 2> $O/final_bench_vlm.err
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none --csv \
  --log-file $O/final_launches.csv python bench.py --steps 1 --warmup 1 --batch-per-rank 16 > $O/final_ncu_ll.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed \
  --cache-control all --clock-control none --csv --log-file $O/final_roof_kd.csv python bench.py --steps 1 --warmup 1 --batch-per-rank 4 > $O/final_ncu_roof.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 1 -c 1 -o $O/final_attn_fwd python scripts/attn_prof.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/final_attn_bwd python scripts/attn_prof.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm2_kernel -s 2 -c 1 -o $O/final_gemm_gu python scripts/gemm_prof.py 32768 11264 2048 fwd > /dev/null 2>&1
ls -la $O/final_*
