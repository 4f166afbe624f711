O=gpurun_out/r44; mkdir -p $O
PMG_DD_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_n2_shared.json 2> $O/bench_n2.err; echo "n2 $?" >> $O/status.txt
timeout 600 python bench.py --steps 20 > $O/bench.json 2> $O/bench.err; echo "n1 $?" >> $O/status.txt
