# Final single-GPU bench lines of every workload (driver-like command lines), with CPU baselines.
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > $O/fb_kd.log 2>&1; echo "== kd $?"; grep '^{' $O/fb_kd.log | cut -c1-200
timeout 1500 python bench.py --workload kd8b --steps 5 --warmup 3 > $O/fb_kd8b.log 2>&1; echo "== kd8b $?"; grep '^{' $O/fb_kd8b.log | cut -c1-200
timeout 900 python bench.py --workload vlm --steps 20 --warmup 5 > $O/fb_vlm.log 2>&1; echo "== vlm $?"; grep '^{' $O/fb_vlm.log | cut -c1-200
timeout 1200 python bench.py --workload section --graph vlm7b --steps 5 --warmup 3 > $O/fb_vlm7b.log 2>&1; echo "== vlm7b $?"; grep '^{' $O/fb_vlm7b.log | cut -c1-200
timeout 1200 python bench.py --workload section --graph omni --steps 5 --warmup 3 > $O/fb_omni.log 2>&1; echo "== omni $?"; grep '^{' $O/fb_omni.log | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/fb_ref.log 2>&1; echo "== ref $?"; grep '^{' $O/fb_ref.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fb_smoke.log 2>&1; echo "== smoke $?"; tail -2 $O/fb_smoke.log
