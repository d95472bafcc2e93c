mkdir -p gpurun_out
timeout 150 python scripts/diag_attn_replay.py capture > gpurun_out/r5c_cap.log 2>&1; echo "== cap $?"; grep -v site-packages gpurun_out/r5c_cap.log | tail -12
timeout 400 python scripts/diag_attn_replay.py all > gpurun_out/r5c_rep.log 2>&1; echo "== rep $?"; cat gpurun_out/r5c_rep.log | tail -12
