O=gpurun_out/r20; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl or sweep or smoother or vcycle or v_cycle" > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
for lib in libpmg_b200.so; do
echo "== $lib" >> $O/qt.log
PMG_B200_LIB=$PWD/paper_2405_19004_b200/$lib timeout 600 python tools/quick_time.py 3 2 6 f64 fused 3 2 7 f64 fused 3 2 8 f64 fused 3 2 6 f32 fused 3 2 7 f32 fused >> $O/qt.log 2>&1
done
echo done >> $O/status.txt
