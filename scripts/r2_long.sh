#!/bin/bash
R=$(pwd)
for rep in 1 2; do
  for v in default base; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> gpurun_out/long.jsonl
    if [ $v = default ]; then (cd scripts && timeout 300 python attn_quick.py >> $R/gpurun_out/long.jsonl 2>&1);
    else (cd scripts && MAESTRO_ATTN_FWD=base timeout 300 python attn_quick.py >> $R/gpurun_out/long.jsonl 2>&1); fi
  done
done
for rep in 1 2; do
  timeout 900 python bench.py --workload kd8b --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-150 >> gpurun_out/long.jsonl
done
timeout 600 python -m pytest tests/test_attention_variants.py tests/test_attention.py -m gpu -q > gpurun_out/long_tests.log 2>&1; echo "rc=$?" >> gpurun_out/long_tests.log
echo done
