set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean > gpurun_out/exp3_tl_dk.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean --opt dk_priv_fixed=60 > gpurun_out/exp3_tl_dk_p60.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 300 --flush clean > gpurun_out/exp3_tl_dk300.txt 2>&1
