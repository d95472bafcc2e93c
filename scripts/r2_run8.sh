mkdir -p gpurun_out
timeout 600 python scripts/parity_report.py > gpurun_out/r8_parity.log 2>&1; echo "== parity $?"; grep -E "^vlm_step|Error" gpurun_out/r8_parity.log | cut -c1-600
DIAG_SECS=2400 timeout 2500 python scripts/diag_hang.py tests -m gpu -p no:randomly > gpurun_out/r8_gputests.log 2>&1; echo "== gpu tests $?"; tail -5 gpurun_out/r8_gputests.log
