O=gpurun_out/r26; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "rhs or gmres or capi" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
timeout 900 python tools/solve_bench.py 1 7 10 3 6 6 7 5 4 > $O/solve_small.jsonl 2>&1; echo "small $?" >> $O/status.txt
timeout 1500 python tools/solve_bench.py > $O/solve.jsonl 2>&1; echo "big $?" >> $O/status.txt
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $O/status.txt
