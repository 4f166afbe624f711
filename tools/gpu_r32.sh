O=gpurun_out/r32; mkdir -p $O
PMG_B200_LIB=$PWD/paper_2405_19004_b200/libpmg_b200_pipe.so timeout 600 python -m pytest tests -m gpu -x -q -k "impl or smoother_variants or sweep" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
bash tools/gpu_ab2.sh r32 "libpmg_b200.so libpmg_b200_pipe.so libpmg_b200_pipe4.so" "3 2 6 f64 fused 3 2 8 f64 fused 3 2 6 f32 fused 3 2 7 f32 fused"
