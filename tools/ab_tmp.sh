O=gpurun_out/ab_wave; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_env_knobs.py -x -q -m gpu > $O/tests.log 2>&1; tail -3 $O/tests.log
for r in 1 2; do for cfg in "0 1" "1 1" "1 2" "1 3"; do set -- $cfg; echo "== MIN_N=$1 BLOCK=$2" >> $O/qt.log
PMG_WAVE_MIN_N=$1 PMG_WAVE_BLOCK=$2 timeout 300 python tools/quick_time.py 3 1 9 f64 fused 3 1 9 f32 fused 3 1 8 f64 fused 3 1 7 f64 fused 3 1 6 f64 fused >> $O/qt.log 2>&1; done; done
