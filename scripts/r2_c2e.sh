#!/bin/bash
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
for rep in 1 2; do
  for v in 1 0; do
    echo "{\"early_head\": $v, \"rep\": $rep}" >> gpurun_out/c2e.jsonl
    MAESTRO_C2_EARLY_HEAD=$v timeout 900 bash -c "$(declare -f tr); tr 2962$v --workload section --graph vlm7b --steps 5 --warmup 3 --no-cpu-baseline" 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'w':'vlm7b','value':d['value'],'loss':d.get('loss')}))" >> gpurun_out/c2e.jsonl
    MAESTRO_C2_EARLY_HEAD=$v timeout 900 bash -c "$(declare -f tr); tr 2963$v --workload section --graph omni --steps 5 --warmup 3 --no-cpu-baseline" 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'w':'omni','value':d['value'],'loss':d.get('loss')}))" >> gpurun_out/c2e.jsonl
  done
done
echo done
