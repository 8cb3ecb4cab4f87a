cd $GRAFT_REPO_ROOT
timeout 300 python tools/rawtrace.py 10 > gpurun_out/r3j_raw.txt 2>&1
for o in 0 262144; do for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --opt dk_slots=$o > gpurun_out/r3j_bench_${o}_$r.json 2>/dev/null; done; done
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "dk_umma or config2" 2>&1 | tail -2 > gpurun_out/r3j_dec.txt
