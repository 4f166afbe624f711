O=gpurun_out/r46; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke $?" >> $O/status.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench $?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref $?" >> $O/status.txt
echo done >> $O/status.txt
