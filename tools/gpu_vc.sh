O=gpurun_out/r07; mkdir -p $O
for cfg in "3 2 6" "3 2 8" "3 4 7" "3 1 9"; do set -- $cfg
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/vc_d$1k$2L$3.csv python tools/prof_target.py $1 $2 $3 f64 fused 0 2 > /dev/null 2>&1
done
echo done >> $O/status.txt
