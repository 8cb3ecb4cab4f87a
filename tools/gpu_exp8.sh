cd $GRAFT_REPO_ROOT
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean > gpurun_out/exp8_tl_dk.txt 2>&1
