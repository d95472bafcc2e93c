mkdir -p gpurun_out
run() { n=$1; s=$2; shift 2
  DIAG_SECS=$s timeout $((s+60)) python scripts/diag_hang.py "$@" > gpurun_out/r7_$n.log 2>&1
  echo "== $n rc=$?"; grep -E "passed|failed|Timeout|Error" gpurun_out/r7_$n.log | tail -3; }
run attn 300 tests/test_attention.py -m gpu
timeout 900 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r7_bench_kd8b.log 2>&1; echo "== kd8b $?"; tail -2 gpurun_out/r7_bench_kd8b.log | cut -c1-1800
timeout 900 python bench.py --workload section --graph vlm7b --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r7_bench_vlm7b.log 2>&1; echo "== vlm7b $?"; tail -2 gpurun_out/r7_bench_vlm7b.log | cut -c1-1800
timeout 900 python bench.py --workload section --graph omni --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r7_bench_omni.log 2>&1; echo "== omni $?"; tail -2 gpurun_out/r7_bench_omni.log | cut -c1-1800
