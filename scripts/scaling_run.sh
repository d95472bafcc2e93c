# One box, N = 1, 2, 4 GPUs back to back: KD (colocated default), KD disjoint, VLM cfg 1 (colocated
# DP default, disjoint section groups), and the
# reference arm; one JSON line per run into gpurun_out/scaling.jsonl.
#   gpurun --gpus 4 -- bash scripts/scaling_run.sh
set -u
OUT=gpurun_out/scaling.jsonl
: > $OUT
run() {  # n, extra args...
  local n=$1; shift
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py "$@" 2>/dev/null | tail -1 >> $OUT
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@" 2>/dev/null | tail -1 >> $OUT
  fi
}
for n in 1 2 4; do run $n; done
for n in 2 4; do run $n --layout disjoint; done
for n in 1 2 4; do run $n --workload vlm; done
for n in 2 4; do run $n --workload vlm --layout disjoint; done
run 1 --impl reference
wc -l $OUT
