#!/usr/bin/env bash
# One gpurun session: GPU parity tests, smoke, bench (default + sweep),
# ncu launch list and one `--set full` capture of the smoother kernel.
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh <tag> [stages]'
# stages (default all): tests smoke bench sweep launches full
set -u
TAG=${1:-r01}
STAGES=${2:-"tests smoke bench sweep launches full"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi -L > "$OUT/gpu.txt" 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' >> "$OUT/gpu.txt"
has() { [[ " $STAGES " == *" $1 "* ]]; }

if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu exit $?" >> "$OUT/status.txt"
fi
if has smoke; then
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/status.txt"
fi
if has bench; then
  timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/status.txt"
fi
if has sweep; then
  for dt in f64 f32; do
    for kl in "1 8" "2 7" "3 7" "4 7" "5 6" "6 6" "7 6"; do
      set -- $kl
      timeout 300 python bench.py --degree $1 --level $2 --dtype $dt --steps 20 --no-cpu \
        >> "$OUT/sweep3d.jsonl" 2>> "$OUT/sweep.err"
    done
  done
  for kl in "1 14" "2 13" "3 12" "4 12" "5 11" "6 11" "7 11"; do
    set -- $kl
    timeout 300 python bench.py --dim 2 --degree $1 --level $2 --dtype f64 --steps 10 --no-cpu \
      >> "$OUT/sweep2d.jsonl" 2>> "$OUT/sweep.err"
  done
  for kl in "2 8" "1 9"; do
    set -- $kl
    timeout 300 python bench.py --dim 3 --degree $1 --level $2 --dtype f64 --steps 10 --no-cpu \
      >> "$OUT/sweep3d_big.jsonl" 2>> "$OUT/sweep.err"
  done
  echo "sweep done" >> "$OUT/status.txt"
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu > "$OUT/launches_bench.log" 2>&1
  echo "launches exit $?" >> "$OUT/status.txt"
fi
if has full; then
  # the headline config: all 8 colour launches of one step (bench roofline.traffic)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:vp_ -s 16 -c 8 \
    -o "$OUT/smooth_d3k2L6f64" python tools/prof_target.py 3 2 6 f64 fused 3 > "$OUT/ncu_c2.log" 2>&1
  for cfg in "3 1 9 f64" "3 2 7 f64" "3 4 7 f64" "3 7 6 f64" "3 4 7 f32" "2 2 13 f64"; do
    set -- $cfg
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:vp_ -s 8 -c 1 \
      -o "$OUT/smooth_d$1k$2L$3$4" python tools/prof_target.py $1 $2 $3 $4 fused 2 > "$OUT/ncu_d$1k$2$4.log" 2>&1
  done
  echo "full exit $?" >> "$OUT/status.txt"
fi
echo done >> "$OUT/status.txt"
