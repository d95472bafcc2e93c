mkdir -p gpurun_out
DIAG_SECS=300 timeout 360 python scripts/diag_hang.py tests/test_gemm.py tests/test_section_compute.py -m gpu > gpurun_out/l2_tests.log 2>&1; echo "== tests $?"; grep -E "passed|failed" gpurun_out/l2_tests.log | tail -1
for h in 0 1 0 1; do
  MAESTRO_GEMM_L2HINT=$h timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/l2_kd_$h.log 2>&1
  grep '^{' gpurun_out/l2_kd_$h.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print('hint=$h', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'), round(d['roofline']['achieved']))"
done
python scripts/gemm_prof.py 32768 11264 2048 swiglu_only > gpurun_out/l2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm2_kernel -s 2 -c 1 --csv \
  python scripts/gemm_prof.py 32768 11264 2048 swiglu_only > gpurun_out/l2_ncu.log 2>&1; grep -E "dram__bytes|duration" gpurun_out/l2_ncu.log | cut -c1-200
