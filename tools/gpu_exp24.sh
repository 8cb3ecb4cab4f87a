cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3 > gpurun_out/exp24_tests.txt
for w in 0 1; do
  timeout 300 python tools/kernel_timeline.py --step 10 --flush clean --opt dk_warm=$w > gpurun_out/exp24_tl_w$w.txt 2>&1
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-extras --opt dk_warm=$w > gpurun_out/exp24_bench_w$w.json 2>/dev/null
done
