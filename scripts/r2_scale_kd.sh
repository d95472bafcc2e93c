# KD (cfg 2) co-located and disjoint at N GPUs with the final code: bash scripts/r2_scale_kd.sh N
N=$1
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 bench.py --gpus $N "${@:2}"; }
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29610 --steps 10 --warmup 3" > gpurun_out/fsc${N}_kd.log 2>&1; echo "== kd colocated N=$N $?"; grep '^{' gpurun_out/fsc${N}_kd.log | cut -c1-200
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29611 --steps 10 --warmup 3 --layout disjoint" > gpurun_out/fsc${N}_kd_dis.log 2>&1; echo "== kd disjoint N=$N $?"; grep '^{' gpurun_out/fsc${N}_kd_dis.log | cut -c1-200
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29612 --workload kd8b --steps 3 --warmup 2" > gpurun_out/fsc${N}_kd8b.log 2>&1; echo "== kd8b colocated N=$N $?"; grep '^{' gpurun_out/fsc${N}_kd8b.log | cut -c1-200
