O=gpurun_out/$1; mkdir -p $O
for lib in $2; do
echo "== $lib" >> $O/qt.log
PMG_B200_LIB=$PWD/paper_2405_19004_b200/$lib timeout 600 python tools/quick_time.py $3 >> $O/qt.log 2>&1
done
echo done >> $O/status.txt
