O=gpurun_out/ab_ls; mkdir -p $O
for r in 1 2; do for lib in libpmg_b200.so libpmg_ls0.so; do echo "== $lib" >> $O/qt.log
PMG_B200_LIB=$PWD/paper_2405_19004_b200/$lib timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 2 6 f64 boundary 3 2 5 f64 fused 3 2 4 f64 fused >> $O/qt.log 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -x -q -m gpu -k "k2 or plane or sweep or C2 or d3k2" > $O/tests.log 2>&1; tail -2 $O/tests.log
