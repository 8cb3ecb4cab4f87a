cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/final/bench_plain_for_ncu.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/final/ncu_launches.log 2>&1
timeout 300 python tools/profile_step.py --step 10 > gpurun_out/final/profile_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dk_kernel -s 10 -c 1 -f -o gpurun_out/final/prof_dk_um_step10 python tools/profile_step.py --step 10 > gpurun_out/final/ncu_full.log 2>&1
