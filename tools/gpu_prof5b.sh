cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:dmma_cp -s 2 -c 1 -o gpurun_out/prof_cp5 -f python tools/time_fused.py 5 128 fused 1 > gpurun_out/prof5b.log 2>&1
