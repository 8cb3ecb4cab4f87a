cd $GRAFT_REPO_ROOT
export CA_LIB=$GRAFT_REPO_ROOT/paper_2402_15220_b200/libchunkattn_debug.so
timeout 1200 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3 > gpurun_out/r2ab_debug_decode.txt
timeout 300 python tools/sanitize_run.py --cfg2 > gpurun_out/r2ab_debug_workloads.txt 2>&1
