cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
H3_DMMA_CFG=0 timeout 600 ncu --set full --import-source on -k regex:sep_fused_dmma3v2 -s 2 -c 1 -o gpurun_out/prof_v2 -f python tools/time_fused.py 3 256 fused 1 > gpurun_out/prof_v2.log 2>&1
H3_DMMA_CFG=6 timeout 600 ncu --set full --import-source on -k regex:sep_fused_dmma3 -s 2 -c 1 -o gpurun_out/prof_v1 -f python tools/time_fused.py 3 256 fused 1 >> gpurun_out/prof_v2.log 2>&1
