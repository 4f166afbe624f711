O=gpurun_out/r25; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "transfer or prolong or restrict or vcycle or v_cycle or fmg or gmres" > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status.txt
for v in 1 0; do
echo "== passes=$v" >> $O/ab.log
PMG_TRANSFER_PASSES=$v timeout 300 python tools/quick_ops.py 3 1 9 f64 3 2 8 f64 3 3 7 f64 3 4 7 f64 3 7 6 f64 3 2 6 f64 3 4 7 f32 >> $O/ab.log 2>&1
PMG_TRANSFER_PASSES=$v timeout 300 python tools/quick_time.py 3 2 6 f64 fused 3 2 8 f64 fused >> $O/ab.log 2>&1
done
echo done >> $O/status.txt
