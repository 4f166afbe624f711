O=gpurun_out/ab_bpf2; mkdir -p $O
for r in 1 2; do for v in 1 0; do echo "== PMG_B_PREFETCH=$v" >> $O/qt.log
PMG_B_PREFETCH=$v timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 3 7 f64 fused 3 3 7 f32 fused 3 4 7 f64 fused 3 4 7 f32 fused 3 5 6 f32 fused 3 3 5 f64 fused >> $O/qt.log 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -x -q -m gpu -k "k3 or k4 or k5 or k6 or pp or d3" > $O/tests.log 2>&1; tail -2 $O/tests.log
