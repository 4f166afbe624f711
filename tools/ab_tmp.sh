O=gpurun_out/ab_gemv; mkdir -p $O
run() { timeout 600 ncu --nvtx --nvtx-include "vc/" --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none --csv --log-file $O/$1.csv python tools/debug/vc_kernels.py $2 > $O/$1.log 2>&1; }
run c2 "3 2 6 f64"; run c2f32 "3 2 6 f32"; run k1 "3 1 6 f64"
timeout 600 python -m pytest tests/test_gpu_coarse_matrix.py tests/test_gpu_dd_capi.py -x -q -m gpu > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 1 6 f64 fused 3 4 5 f64 fused > $O/qt.log 2>&1
