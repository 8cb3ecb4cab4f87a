cd $GRAFT_REPO_ROOT
for o in 0 512 1024 1536; do
timeout 300 python tools/rawtrace.py 10 dk_slots=$o > gpurun_out/r2z_$o.txt 2>&1
done
