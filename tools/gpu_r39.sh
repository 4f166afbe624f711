O=gpurun_out/r39; mkdir -p $O
PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_b200_pk3.so timeout 600 python -m pytest tests -m gpu -x -q -k "impl" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_b200_pk3.so PMG_IMPLS=auto,plane timeout 600 python tools/quick_time.py 3 3 6 f64 fused 3 3 7 f64 fused 3 3 6 f32 fused 3 3 7 f32 fused > $O/qt.log 2>&1
echo done >> $O/status.txt
