O=gpurun_out/ab_cm; mkdir -p $O
for r in 1 2; do for n in 1331 3375; do echo "== $n" >> $O/qt.log
PMG_COARSE_MAT_N=$n timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 1 6 f64 fused 3 4 5 f64 fused 3 2 7 f64 fused 3 4 6 f32 fused >> $O/qt.log 2>&1; done; done
for n in 1331 3375; do PMG_COARSE_MAT_N=$n timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu > $O/bench_$n.json 2> $O/bench_$n.err; done
PMG_COARSE_MAT_N=3375 timeout 900 python -m pytest tests/ -x -q -m gpu -k "vcycle or v_cycle or coarse or fmg or dd or gmres" > $O/tests.log 2>&1; tail -3 $O/tests.log
