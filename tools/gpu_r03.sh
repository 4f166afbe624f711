mkdir -p gpurun_out/r03
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r03/pytest_gpu.log 2>&1; echo "pytest $?" >> gpurun_out/r03/status.txt
PMG_IMPLS=auto,plane timeout 600 python tools/quick_time.py 3 1 8 f64 fused 3 1 9 f64 fused 3 1 8 f32 fused 2 1 12 f64 fused 2 1 14 f64 fused > gpurun_out/r03/qt.log 2>&1; echo "qt $?" >> gpurun_out/r03/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vp_point -s 8 -c 1 -o gpurun_out/r03/point_d3k1L9f64 python tools/prof_target.py 3 1 9 f64 fused 2 > /dev/null 2>&1
echo done >> gpurun_out/r03/status.txt
