O=gpurun_out/r41; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
PMG_DD_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_n2_shared.json 2> $O/bench_n2.err; echo "n2 $?" >> $O/status.txt
timeout 600 python bench.py --dtype f32 --steps 20 > $O/bench_f32.json 2> $O/bench_f32.err; echo "f32 $?" >> $O/status.txt
echo done >> $O/status.txt
