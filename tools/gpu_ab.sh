# A/B of alternative builds: bash tools/gpu_ab.sh TAG "lib1 lib2 ..." "quick_time args"
O=gpurun_out/$1; mkdir -p $O
for lib in $2; do
  echo "== $lib" >> $O/ab.log
  PMG_B200_LIB=$PWD/paper_2405_19004_b200/$lib timeout 300 python tools/quick_time.py $3 >> $O/ab.log 2>&1
done
echo done >> $O/status.txt
