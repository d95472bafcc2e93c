# one compute-sanitizer tool per gpurun call (B200_PROFILING.md); usage: bash scripts/r2_sanitize.sh <tool>
mkdir -p gpurun_out
tool=$1
python scripts/sanitize_driver.py all > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/san_plain.log; exit 1; }
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_driver.py all > gpurun_out/san_$tool.log 2>&1
echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK|ok all|Error|Hazard" gpurun_out/san_$tool.log | head -20
