#!/bin/bash
timeout 400 python -m pytest tests/test_attention.py tests/test_attention_variants.py tests/test_graph_exec.py -m gpu -q -x > gpurun_out/a9_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/a9_tests.log
(cd scripts && timeout 300 python attn_quick.py > ../gpurun_out/a9_quick.jsonl 2>&1)
timeout 900 python bench.py --workload section --graph vlm7b --steps 5 --warmup 3 > gpurun_out/a9_vlm7b.log 2>&1
echo done
