#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/b1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b1_tests.log
timeout 600 python bench.py > gpurun_out/b1_bench_kd.json 2> gpurun_out/b1_bench_kd.err
timeout 900 python bench.py --workload kd8b > gpurun_out/b1_bench_kd8b.json 2> gpurun_out/b1_bench_kd8b.err
echo done
