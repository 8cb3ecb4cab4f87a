cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py --cfg2 > gpurun_out/sanitizer/memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/memcheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/synccheck.txt
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/racecheck.txt
