cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/r3o_t.txt
timeout 600 python bench_sweep.py --points cfg5 > gpurun_out/r3o_cfg5.txt 2>&1
timeout 600 python bench_prefill.py > gpurun_out/r3o_prefill.txt 2>&1
