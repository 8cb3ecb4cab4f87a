cd $GRAFT_REPO_ROOT; ./tools/dsmem_probe > gpurun_out/exp13_dsmem.txt 2>&1
