cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dk_kernel -s 10 -c 1 -o gpurun_out/dk_step10 -f python tools/profile_step.py --step 12 > gpurun_out/exp14.log 2>&1
ncu -i gpurun_out/dk_step10.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/dk_step10_src.csv 2>/dev/null
ncu -i gpurun_out/dk_step10.ncu-rep --page raw --csv > gpurun_out/dk_step10_raw.csv 2>/dev/null
ncu -i gpurun_out/dk_step10.ncu-rep --page details --csv > gpurun_out/dk_step10_details.csv 2>/dev/null
ls -la gpurun_out/dk_step10*
