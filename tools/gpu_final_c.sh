cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/final/sanitizer_racecheck.txt 2>&1
