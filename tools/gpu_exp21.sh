cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/synccheck.txt
