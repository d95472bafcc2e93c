mkdir -p gpurun_out
for cg in 4; do
  MAESTRO_ATTN_CG=$cg DIAG_SECS=200 timeout 260 python scripts/diag_hang.py tests/test_attention.py -m gpu > gpurun_out/cg${cg}_tests.log 2>&1
  echo "== cg$cg tests $?"; grep -E "passed|failed|Timeout" gpurun_out/cg${cg}_tests.log | tail -2
  MAESTRO_ATTN_CG=$cg timeout 300 python scripts/attn_h2h.py > gpurun_out/cg${cg}_h2h.log 2>&1
  echo "== cg$cg h2h"; grep '^{' gpurun_out/cg${cg}_h2h.log | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], round(d['ours_fwd_tflops']), round(d.get('cudnn_fwd_tflops',0)))"
done
