# C2 experiments on one box: bash scripts/r2_c2.sh <N>
mkdir -p gpurun_out
N=$1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 scripts/nccl_bw.py > gpurun_out/c2_nccl_$N.log 2>&1; echo "== nccl"; grep '^{' gpurun_out/c2_nccl_$N.log
for ov in 0 1; do
  MAESTRO_C2_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$ov bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/c2_kd_${N}_$ov.log 2>&1
  echo "== kd overlap=$ov"; grep '^{' gpurun_out/c2_kd_${N}_$ov.log | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2), d['ms_per_step'], d.get('grad_allreduce'))"
  MAESTRO_C2_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$ov bench.py --gpus $N --workload section --graph vlm7b --steps 3 --warmup 2 > gpurun_out/c2_vlm7b_${N}_$ov.log 2>&1
  echo "== vlm7b overlap=$ov"; grep '^{' gpurun_out/c2_vlm7b_${N}_$ov.log | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2), d['ms_per_step'])"
done
