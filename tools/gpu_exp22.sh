cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2/pytest_gpu.txt
timeout 600 python bench_serve.py > gpurun_out/r2/serve.jsonl 2> gpurun_out/r2/serve.err
timeout 600 python bench_prefill.py > gpurun_out/r2/prefill.jsonl 2> gpurun_out/r2/prefill.err
timeout 900 python bench_sweep.py --points all > gpurun_out/r2/sweep.jsonl 2> gpurun_out/r2/sweep.err
