cd $GRAFT_REPO_ROOT
./tools/launch_probe > gpurun_out/exp11_launch_probe.txt 2>&1
