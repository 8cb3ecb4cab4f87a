cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:dk_kernel -c 30 --csv --log-file gpurun_out/exp10_ncu.csv python tools/profile_step.py --step 40 > gpurun_out/exp10.log 2>&1
