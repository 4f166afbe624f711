O=gpurun_out/r35; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl or smoother_variants or vcycle or fmg" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_IMPLS=line,auto timeout 600 python tools/quick_time.py 2 2 10 f64 fused 2 2 13 f64 fused 2 2 13 f32 fused 2 3 12 f64 fused 2 3 12 f32 fused > $O/qt.log 2>&1
echo done >> $O/status.txt
