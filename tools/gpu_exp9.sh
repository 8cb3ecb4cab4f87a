cd $GRAFT_REPO_ROOT
timeout 300 python tools/launch_overhead.py > gpurun_out/exp9_launch.txt 2>&1
