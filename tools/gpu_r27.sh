O=gpurun_out/r27; mkdir -p $O
timeout 1500 python tools/solve_bench.py > $O/solve.jsonl 2>&1; echo "big $?" >> $O/status.txt
