mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_attention.py -x -q -m gpu -k "hd128" 2>&1 | tail -30 > gpurun_out/r1_attn128.log
tail -5 gpurun_out/r1_attn128.log
timeout 900 python -m pytest tests/test_attention.py tests/test_gemm.py tests/test_section_compute.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r1_tests.log
tail -5 gpurun_out/r1_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_kd.log 2>&1; tail -3 gpurun_out/r1_bench_kd.log
timeout 900 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r1_bench_kd8b.log 2>&1; tail -5 gpurun_out/r1_bench_kd8b.log
