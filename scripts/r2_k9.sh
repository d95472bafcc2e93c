mkdir -p gpurun_out
for r in 4 1; do echo "== rows/SM $r"; MAESTRO_KD_ROWS_PER_SM=$r timeout 200 python scripts/kd_loss_bench.py; done
DIAG_SECS=200 timeout 260 python scripts/diag_hang.py tests/test_section_compute.py -m gpu -k kd_loss > gpurun_out/k9_tests.log 2>&1; echo "== tests $?"; grep -E "passed|failed" gpurun_out/k9_tests.log | tail -1
