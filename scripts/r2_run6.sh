mkdir -p gpurun_out
timeout 600 python scripts/parity_report.py > gpurun_out/r6_parity.log 2>&1; echo "== parity $?"; tail -8 gpurun_out/r6_parity.log | cut -c1-700
timeout 600 python scripts/attn_h2h.py > gpurun_out/r6_h2h.log 2>&1; echo "== h2h $?"; tail -8 gpurun_out/r6_h2h.log | cut -c1-500
