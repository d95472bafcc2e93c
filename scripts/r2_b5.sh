#!/bin/bash
timeout 300 python -m pytest tests/test_section_compute.py -m gpu -q -x -k "ce_loss or kd_loss" > gpurun_out/b5_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b5_tests.log
timeout 300 python -m pytest tests/test_graph_exec.py tests/test_vlm.py -m gpu -q -x > gpurun_out/b5_tests2.log 2>&1
echo "tests rc=$?" >> gpurun_out/b5_tests2.log
timeout 900 python bench.py --workload section --graph vlm7b --steps 5 --warmup 3 > gpurun_out/b5_vlm7b.log 2>&1
echo done
