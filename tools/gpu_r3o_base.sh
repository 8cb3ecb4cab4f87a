cd $GRAFT_REPO_ROOT
timeout 600 python bench_sweep.py --points cfg5 > gpurun_out/r3o_cfg5_base.txt 2>&1
timeout 600 python bench_prefill.py > gpurun_out/r3o_prefill_base.txt 2>&1
