cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/exp18_suite.txt
timeout 300 python bench.py --steps 10 --warmup 3 --workload cfg5 --no-extras --no-cpu > gpurun_out/exp18_cfg5_w1.json 2> gpurun_out/exp18_cfg5_w1.err
