#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pg_tests.log
timeout 300 python scripts/plan_bench.py > gpurun_out/pg_plan.jsonl 2>&1
timeout 600 python bench.py > gpurun_out/pg_bench.json 2>gpurun_out/pg_bench.err
echo done
