cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2 > gpurun_out/r3m_dec.txt
timeout 300 python tools/rawtrace.py 10 > gpurun_out/r3m_raw.txt 2>&1
for r in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/r3m_bench_$r.json 2>/dev/null; done
