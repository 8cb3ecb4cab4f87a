set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
i=0
for o in "" "--opt cf_splits=4" "--opt cf_splits=3" "--opt cf_splits=2" "--opt cf_splits=4 --opt cf_unit_cost=10" "--opt fused=0"; do
  i=$((i+1))
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu $o > gpurun_out/exp1_v$i.json 2> gpurun_out/exp1_v$i.err
  echo "$o" > gpurun_out/exp1_v$i.opt
done
timeout 300 python tools/kernel_timeline.py --step 5 --flush clean > gpurun_out/exp1_tl_default.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 5 --flush clean --opt cf_splits=4 > gpurun_out/exp1_tl_s4.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 5 --flush clean --opt cf_splits=2 > gpurun_out/exp1_tl_s2.txt 2>&1
