set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -30 > gpurun_out/exp2_decode_tests.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/exp2_bench.json 2> gpurun_out/exp2_bench.err
tail -5 gpurun_out/exp2_bench.err
