#!/bin/bash
timeout 600 python -m pytest tests/test_attention_variants.py tests/test_attention.py -m gpu -q -x > gpurun_out/b4_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b4_tests.log
if grep -q "tests rc=0" gpurun_out/b4_tests.log; then
  MAESTRO_ATTN_FWD=dec timeout 60 python scripts/diag_dec.py both > gpurun_out/b4_diag.log 2>&1
  timeout 600 python bench.py > gpurun_out/b4_bench_kd.json 2> gpurun_out/b4_bench_kd.err
fi
echo done
