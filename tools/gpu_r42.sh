O=gpurun_out/r43; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl or smoother_variants" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_IMPLS=plane,patch,patch3 timeout 600 python tools/quick_time.py 3 2 6 f64 fused 3 2 7 f64 fused 3 2 8 f64 fused 3 2 6 f32 fused 3 2 7 f32 fused > $O/qt.log 2>&1
echo done >> $O/status.txt
