cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -15 > gpurun_out/exp4_decode_tests.txt
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean > gpurun_out/exp4_tl_dk.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 300 --flush clean > gpurun_out/exp4_tl_dk300.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/exp4_bench.json 2> gpurun_out/exp4_bench.err
