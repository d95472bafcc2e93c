mkdir -p gpurun_out
timeout 600 python scripts/parity_report.py > gpurun_out/r6_parity.log 2>&1; echo "== parity $?"; tail -8 gpurun_out/r6_parity.log | cut -c1-600
timeout 600 python scripts/attn_h2h.py > gpurun_out/r6_h2h.log 2>&1; echo "== h2h $?"; tail -8 gpurun_out/r6_h2h.log | cut -c1-500
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  for w in attn gemm kd handoff plan; do
    timeout 600 $CS --tool $tool --print-limit 20 python scripts/sanitize_driver.py $w > gpurun_out/r6_san_${tool}_$w.log 2>&1
    echo "== $tool $w rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok |Error" gpurun_out/r6_san_${tool}_$w.log | head -4
  done
done
