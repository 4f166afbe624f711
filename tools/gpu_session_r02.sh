#!/usr/bin/env bash
# One gpurun session (round 2): GPU tests, smoke, bench (headline + sweeps),
# C2 kernel-organisation A/B, the timed step's DRAM traffic (application
# replay) and the ncu launch list of the bench command.
#   gpurun --timeout 3000 -- 'bash tools/gpu_session_r02.sh <tag> [stages]'
# stages (default all): tests smoke bench ab traffic launches full
set -u
TAG=${1:-r02}
STAGES=${2:-"tests smoke bench ab traffic launches"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi -L > "$OUT/gpu.txt" 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' >> "$OUT/gpu.txt"
free -g >> "$OUT/gpu.txt"
has() { [[ " $STAGES " == *" $1 "* ]]; }

if has tests; then
  timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu exit $?" >> "$OUT/status.txt"
fi
if has smoke; then
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/status.txt"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/status.txt"
fi
if has ab; then
  PMG_IMPLS=plane,patch,line,sweep timeout 600 python tools/quick_time.py 3 2 6 f64 fused 3 2 6 f32 fused \
    > "$OUT/ab_c2_impls.txt" 2>&1
  echo "ab exit $?" >> "$OUT/status.txt"
fi
if has traffic; then
  timeout 900 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:vp_ -c 64 --csv \
    --log-file "$OUT/step_traffic_c2.csv" python bench.py --steps 3 --warmup 3 --no-cpu --no-sweep \
    > "$OUT/step_traffic_bench.log" 2>&1
  echo "traffic exit $?" >> "$OUT/status.txt"
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu --no-sweep \
    > "$OUT/launches_bench.log" 2>&1
  echo "launches exit $?" >> "$OUT/status.txt"
fi
if has full; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:vp_ -s 16 -c 8 \
    -o "$OUT/smooth_d3k2L6f64" python tools/prof_target.py 3 2 6 f64 fused 3 > "$OUT/ncu_c2.log" 2>&1
  echo "full exit $?" >> "$OUT/status.txt"
fi
echo done >> "$OUT/status.txt"
