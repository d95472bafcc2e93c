mkdir -p gpurun_out
run() {  # name, watchdog seconds, pytest args...
  n=$1; s=$2; shift 2
  DIAG_SECS=$s timeout $((s+60)) python scripts/diag_hang.py "$@" > gpurun_out/r4_$n.log 2>&1
  echo "== $n rc=$?"; grep -E "passed|failed|Timeout|Error" gpurun_out/r4_$n.log | tail -3
}
run sc 400 tests/test_section_compute.py -m gpu
run gx 400 tests/test_graph_exec.py -m gpu
run pu 200 tests/test_parallel_upstream.py tests/test_handoff.py -m gpu
run gemm 300 tests/test_gemm.py -m gpu
timeout 900 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r4_bench_kd8b.log 2>&1; tail -2 gpurun_out/r4_bench_kd8b.log | cut -c1-1500
timeout 900 python bench.py --workload section --graph vlm7b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r4_bench_vlm7b.log 2>&1; tail -2 gpurun_out/r4_bench_vlm7b.log | cut -c1-1500
