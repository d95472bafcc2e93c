mkdir -p gpurun_out
for f in test_handoff test_graph_exec test_vlm test_section_compute test_attention test_gemm; do
  timeout 900 python -m pytest tests/$f.py -q -m gpu --timeout 300 -x 2>&1 | tail -40 > gpurun_out/r2_$f.log
  echo "== $f"; tail -3 gpurun_out/r2_$f.log
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_kd.log 2>&1; tail -2 gpurun_out/r2_bench_kd.log | cut -c1-600
timeout 900 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_kd8b.log 2>&1; tail -2 gpurun_out/r2_bench_kd8b.log | cut -c1-600
