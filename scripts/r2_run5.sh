mkdir -p gpurun_out
DIAG_SECS=200 timeout 260 python scripts/diag_kd8b.py attn > gpurun_out/r5_attn.log 2>&1; echo "== attn $?"; tail -45 gpurun_out/r5_attn.log | grep -v "site-packages"
DIAG_SECS=300 timeout 360 python scripts/diag_kd8b.py kd8b > gpurun_out/r5_kd8b.log 2>&1; echo "== kd8b $?"; tail -45 gpurun_out/r5_kd8b.log | grep -v "site-packages"
DIAG_SECS=300 timeout 360 python scripts/diag_kd8b.py vlm7b > gpurun_out/r5_vlm7b.log 2>&1; echo "== vlm7b $?"; tail -45 gpurun_out/r5_vlm7b.log | grep -v "site-packages"
