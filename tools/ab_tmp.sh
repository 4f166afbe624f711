O=gpurun_out/ab_pers; mkdir -p $O
PMG_PLANE_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sweep_bitwise or d3k2 or plane" > $O/tests.log 2>&1; tail -2 $O/tests.log
for r in 1 2; do
echo "== base" >> $O/qt.log; timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 2 5 f64 fused >> $O/qt.log 2>&1
for tpc in 0 -1 2 3; do echo "== persist tpc=$tpc" >> $O/qt.log; PMG_PLANE_PERSIST=1 PMG_PLANE_PERSIST_TPC=$tpc timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused 3 2 5 f64 fused >> $O/qt.log 2>&1; done; done
