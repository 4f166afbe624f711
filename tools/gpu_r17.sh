O=gpurun_out/r17; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_IMPLS=line,auto timeout 600 python tools/quick_time.py 3 3 7 f64 fused 3 4 7 f64 fused 3 5 6 f64 fused 3 3 7 f32 fused 3 4 7 f32 fused 3 5 6 f32 fused > $O/qt.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:vp_smooth -s 8 -c 1 -o $O/pp_d3k4L7f64 python tools/prof_target.py 3 4 7 f64 fused 2 > /dev/null 2>&1
echo done >> $O/status.txt
