mkdir -p gpurun_out
export CUDA_LAUNCH_BLOCKING=1
LAYERS=1 DIAG_SECS=120 timeout 180 python scripts/diag_kd8b.py kd8b > gpurun_out/r5b_kd8b.log 2>&1; echo "== kd8b $?"; tail -30 gpurun_out/r5b_kd8b.log | grep -v "site-packages"
LAYERS=1 DIAG_SECS=120 timeout 180 python scripts/diag_kd8b.py vlm7b > gpurun_out/r5b_vlm7b.log 2>&1; echo "== vlm7b $?"; tail -30 gpurun_out/r5b_vlm7b.log | grep -v "site-packages"
