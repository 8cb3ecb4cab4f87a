cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "config2 or dk_umma" 2>&1 | tail -2 > gpurun_out/r3b_dec.txt
timeout 300 python tools/rawtrace.py 10 > gpurun_out/r3b_raw.txt 2>&1
timeout 300 python tools/rawtrace.py 10 dk_slots=16384 > gpurun_out/r3b_raw2d.txt 2>&1
for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/r3b_bench_$r.json 2>/dev/null;
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --opt dk_slots=16384 > gpurun_out/r3b_bench2d_$r.json 2>/dev/null; done
