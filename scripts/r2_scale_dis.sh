# disjoint-layout runs only: bash scripts/r2_scale_dis.sh <N>
mkdir -p gpurun_out
N=$1
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 bench.py --gpus $N "${@:2}"; }
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29511 --steps 10 --warmup 3 --layout disjoint" > gpurun_out/sc${N}_kd_dis.log 2>&1; echo "== kd disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_kd_dis.log | cut -c1-300
timeout 1200 bash -c "$(declare -f tr); N=$N; tr 29512 --workload kd8b --steps 3 --warmup 2 --layout disjoint" > gpurun_out/sc${N}_kd8b_dis.log 2>&1; echo "== kd8b disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_kd8b_dis.log | cut -c1-300
timeout 600 bash -c "$(declare -f tr); N=$N; tr 29517 --workload vlm --layout disjoint --steps 20 --warmup 5" > gpurun_out/sc${N}_vlm_dis.log 2>&1; echo "== vlm disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_vlm_dis.log | cut -c1-300
