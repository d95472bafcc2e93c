#!/bin/bash
# final verification: the driver's GPU tiers twice (flakiness), smoke, default bench
for rep in 1 2; do
  timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fc_tests_$rep.log 2>&1; echo "tests $rep rc=$?" >> gpurun_out/fc_summary.log
  tail -1 gpurun_out/fc_tests_$rep.log >> gpurun_out/fc_summary.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fc_summary.log
timeout 600 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?" >> gpurun_out/fc_summary.log
timeout 600 python bench.py --impl reference > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo "ref rc=$?" >> gpurun_out/fc_summary.log
