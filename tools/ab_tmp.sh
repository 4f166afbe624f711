O=gpurun_out/ab_rpar; mkdir -p $O
timeout 1200 python -m pytest tests/ -x -q -m gpu -k "transfer or restrict or vcycle or dd or slab or fmg or gmres or coarse" > $O/tests.log 2>&1; tail -2 $O/tests.log
run() { timeout 600 ncu --nvtx --nvtx-include "vc/" --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none --csv --log-file $O/$1.csv python tools/debug/vc_kernels.py $2 > $O/$1.log 2>&1; }
run c2 "3 2 6 f64"; run k1 "3 1 8 f64"; run k3 "3 3 6 f64"; run k4 "3 4 6 f64"
for r in 1 2; do for v in 1 0; do echo "== PMG_RESTRICT_PAR=$v" >> $O/qt.log
PMG_RESTRICT_PAR=$v timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 1 8 f64 fused 3 3 6 f64 fused 3 4 6 f64 fused 3 3 7 f32 fused >> $O/qt.log 2>&1; done; done
