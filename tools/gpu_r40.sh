O=gpurun_out/r40; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "impl or operator" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
for lib in libpmg_b200.so libpmg_b200_ty4.so libpmg_b200_ty16.so; do
echo "== $lib" >> $O/ab.log
PMG_B200_LIB=$PWD/paper_2405_19004_b200/$lib timeout 300 python tools/quick_ops.py 3 1 9 f64 3 2 8 f64 3 3 7 f64 3 4 7 f64 3 7 6 f64 3 2 6 f64 >> $O/ab.log 2>&1
done
echo done >> $O/status.txt
