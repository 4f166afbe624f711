O=gpurun_out/r36; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl or smoother_variants" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_IMPLS=plane,patch timeout 600 python tools/quick_time.py 3 2 6 f64 fused 3 2 7 f64 fused 3 2 8 f64 fused 3 2 6 f32 fused 3 2 7 f32 fused > $O/qt.log 2>&1
PMG_IMPL=patch timeout 300 ncu --set full --clock-control none --import-source on -k regex:vp_patch3d -s 8 -c 1 -o $O/patch3d_d3k2L6f64 python tools/prof_target.py 3 2 6 f64 fused 2 > /dev/null 2>&1
echo done >> $O/status.txt
