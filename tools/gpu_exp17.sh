cd $GRAFT_REPO_ROOT
( time timeout 600 python bench.py --steps 20 --warmup 5 ) > gpurun_out/exp17_bench.json 2> gpurun_out/exp17_bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --workload cfg5 > gpurun_out/exp17_cfg5_w1.json 2> gpurun_out/exp17_cfg5_w1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --dist-backend gloo > gpurun_out/exp17_cfg5_w2.json 2> gpurun_out/exp17_cfg5_w2.err
