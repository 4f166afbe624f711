O=gpurun_out/ab_cb2; mkdir -p $O
run() { timeout 600 ncu --nvtx --nvtx-include "vc/" --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none --csv --log-file $O/$1.csv python tools/debug/vc_kernels.py $2 > $O/$1.log 2>&1; }
for lib in b200 mb6 fly flymb6 nw8; do for c in 4 8; do
PMG_OP_CB_CTAS=$c PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_$lib.so run ${lib}_c${c}_c2 "3 2 6 f64"
PMG_OP_CB_CTAS=$c PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_$lib.so run ${lib}_c${c}_k2L7 "3 2 7 f64"
PMG_OP_CB_CTAS=$c PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_$lib.so run ${lib}_c${c}_f32 "3 2 6 f32"
done; done
