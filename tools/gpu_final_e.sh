cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench2.json 2> gpurun_out/final/bench2.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/final/bench_plain2.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dk_kernel -c 200 --csv --log-file gpurun_out/final/launches_dk.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/final/ncu_launches_dk.log 2>&1
