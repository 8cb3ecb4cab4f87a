cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/final/smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/final/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 300 python tools/sanitize_run.py --cfg2 > gpurun_out/final/sanitize_plain.txt 2>&1
timeout 300 python tools/kernel_timeline.py --step 10 --flush clean > gpurun_out/final/timeline_step10.txt 2>&1
timeout 300 python tools/rawtrace.py 10 > gpurun_out/final/rawtrace_step10.txt 2>&1
