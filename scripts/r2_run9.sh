mkdir -p gpurun_out
DIAG_SECS=900 timeout 960 python scripts/diag_hang.py tests -m gpu > gpurun_out/r9_gputests.log 2>&1; echo "== gpu tests $?"; tail -3 gpurun_out/r9_gputests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r9_kd.log 2>&1; echo "== kd $?"; grep '^{' gpurun_out/r9_kd.log | cut -c1-300
timeout 600 python bench.py --workload vlm --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r9_vlm.log 2>&1; echo "== vlm $?"; grep '^{' gpurun_out/r9_vlm.log | cut -c1-300
