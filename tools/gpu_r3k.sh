cd $GRAFT_REPO_ROOT
for v in 2 3 4; do for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --opt dk_slots=$((32768*v)) > gpurun_out/r3k_v${v}_$r.json 2>/dev/null; done; done
