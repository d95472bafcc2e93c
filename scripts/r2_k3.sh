mkdir -p gpurun_out
DIAG_SECS=300 timeout 360 python scripts/diag_hang.py tests/test_device_scheduler.py tests/test_parallel_upstream.py -m gpu > gpurun_out/k3_tests.log 2>&1; echo "== tests $?"; grep -E "passed|failed|Timeout" gpurun_out/k3_tests.log | tail -2
timeout 300 python scripts/plan_bench.py > gpurun_out/k3_plan.log 2>&1; echo "== plan"; cat gpurun_out/k3_plan.log | tail -6
