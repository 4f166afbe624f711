mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest $?" >> gpurun_out/r02/status.txt
PMG_IMPLS=line,plane timeout 600 python tools/quick_time.py 3 1 8 f64 fused 3 2 6 f64 fused 3 2 7 f64 fused 3 3 7 f64 fused 3 1 8 f32 fused 3 2 7 f32 fused 3 3 7 f32 fused > gpurun_out/r02/qt.log 2>&1; echo "qt $?" >> gpurun_out/r02/status.txt
for k in 1 2 3; do L=$((k==1?8:(k==2?6:7))); timeout 300 ncu --set full --clock-control none --import-source on -k regex:vp_smooth -s 8 -c 1 -o gpurun_out/r02/plane_d3k${k}L${L}f64 python tools/prof_target.py 3 $k $L f64 fused 2 > /dev/null 2>&1; done
echo done >> gpurun_out/r02/status.txt
