cd $GRAFT_REPO_ROOT
for qq in 0 64 128 256 512; do
  for o in "dk=1" "dk=0"; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --question $qq --opt $o > gpurun_out/exp15_q${qq}_${o}.json 2>/dev/null
  done
done
for nsh in 0 1024; do
  for o in "dk=1" "dk=0"; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --n-shared $nsh --question 1024 --opt $o > gpurun_out/exp15_ns${nsh}_${o}.json 2>/dev/null
  done
done
