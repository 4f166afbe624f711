O=gpurun_out/r23; mkdir -p $O
for t in 0 64 256 1024 4096; do
echo "== tiles $t" >> $O/qt.log
PMG_SWEEP_AUTO_TILES=$t timeout 600 python tools/quick_time.py 3 2 6 f64 fused 3 2 8 f64 fused 3 2 6 f32 fused >> $O/qt.log 2>&1
done
echo done >> $O/status.txt
