cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2 > gpurun_out/exp23_tests.txt
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean > gpurun_out/exp23_tl.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/exp23_bench.json 2>/dev/null
