cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:recon_sep -s 1 -c 1 -o gpurun_out/prof_recon5 -f python tools/time_fused.py 5 128 two_pass 1 > gpurun_out/prof5.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:sep_fused_kernel -s 1 -c 1 -o gpurun_out/prof_fused5 -f python tools/time_fused.py 5 128 fused 1 >> gpurun_out/prof5.log 2>&1
