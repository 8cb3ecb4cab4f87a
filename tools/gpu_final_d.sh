cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/final/sanitizer_synccheck.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/final/sanitizer_memcheck.txt 2>&1
