# multi-GPU runs on one box: bash scripts/r2_scale.sh <N>
mkdir -p gpurun_out
N=$1
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 bench.py --gpus $N "${@:2}"; }
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29510 --steps 10 --warmup 3" > gpurun_out/sc${N}_kd.log 2>&1; echo "== kd colocated N=$N $?"; grep '^{' gpurun_out/sc${N}_kd.log | cut -c1-300
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29511 --steps 10 --warmup 3 --layout disjoint" > gpurun_out/sc${N}_kd_dis.log 2>&1; echo "== kd disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_kd_dis.log | cut -c1-300
timeout 1200 bash -c "$(declare -f tr); N=$N; tr 29512 --workload kd8b --steps 3 --warmup 2 --layout disjoint" > gpurun_out/sc${N}_kd8b_dis.log 2>&1; echo "== kd8b disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_kd8b_dis.log | cut -c1-300
timeout 1200 bash -c "$(declare -f tr); N=$N; tr 29513 --workload kd8b --steps 3 --warmup 2" > gpurun_out/sc${N}_kd8b.log 2>&1; echo "== kd8b colocated N=$N $?"; grep '^{' gpurun_out/sc${N}_kd8b.log | cut -c1-300
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29514 --workload section --graph vlm7b --steps 3 --warmup 2" > gpurun_out/sc${N}_vlm7b.log 2>&1; echo "== vlm7b N=$N $?"; grep '^{' gpurun_out/sc${N}_vlm7b.log | cut -c1-300
timeout 900 bash -c "$(declare -f tr); N=$N; tr 29515 --workload section --graph omni --steps 3 --warmup 2" > gpurun_out/sc${N}_omni.log 2>&1; echo "== omni N=$N $?"; grep '^{' gpurun_out/sc${N}_omni.log | cut -c1-300
timeout 600 bash -c "$(declare -f tr); N=$N; tr 29516 --workload vlm --steps 20 --warmup 5" > gpurun_out/sc${N}_vlm.log 2>&1; echo "== vlm N=$N $?"; grep '^{' gpurun_out/sc${N}_vlm.log | cut -c1-300
timeout 600 bash -c "$(declare -f tr); N=$N; tr 29517 --workload vlm --layout disjoint --steps 20 --warmup 5" > gpurun_out/sc${N}_vlm_dis.log 2>&1; echo "== vlm disjoint N=$N $?"; grep '^{' gpurun_out/sc${N}_vlm_dis.log | cut -c1-300
