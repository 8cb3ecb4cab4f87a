cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2 > gpurun_out/r3l_dec.txt
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config4 or config3" 2>&1 | tail -2 > gpurun_out/r3l_cfg.txt
timeout 300 python tools/rawtrace.py 10 > gpurun_out/r3l_raw.txt 2>&1
for o in 0 1048576; do for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --opt dk_slots=$o > gpurun_out/r3l_bench_${o}_$r.json 2>/dev/null; done; done
