#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x -k "vlm or graph or plan or sched" > gpurun_out/vg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/vg_tests.log
timeout 600 python bench.py --workload vlm --steps 20 --warmup 5 > gpurun_out/vg_vlm.log 2>&1
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
timeout 600 bash -c "$(declare -f tr); tr 29517 --workload vlm --layout disjoint --steps 20 --warmup 5" > gpurun_out/vg_vlm_dis.log 2>&1; echo "dis rc=$?" >> gpurun_out/vg_tests.log
echo done
