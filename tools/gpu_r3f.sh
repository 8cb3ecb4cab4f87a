cd $GRAFT_REPO_ROOT
for v in 3 4 5; do
timeout 300 python tools/rawtrace.py 10 dk_slots=$((32768*v)) > gpurun_out/r3f_v$v.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --opt dk_slots=$((32768*v)) > gpurun_out/r3f_bench_v$v.json 2>/dev/null
done
