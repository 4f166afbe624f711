O=gpurun_out/r37; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_IMPLS=plane,patch timeout 600 python tools/quick_time.py 3 3 6 f32 fused 3 3 7 f32 fused > $O/qt.log 2>&1

echo done >> $O/status.txt
