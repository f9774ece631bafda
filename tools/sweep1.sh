cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for c in 0 1 2 3 4 5; do for cy in 1 2; do H3_DMMA_CFG=$c H3_DMMA_CLUSTER_Y=$cy timeout 200 python tools/time_fused.py 3 512 fused 6; done; done
H3_FUSED_IMPL=dfma timeout 200 python tools/time_fused.py 3 512 fused 4
timeout 600 python tools/time_fused.py 3 512 two_pass 2
timeout 300 python tools/time_fused.py 3 256 two_pass 4
timeout 300 python tools/time_fused.py 5 256 fused 4
timeout 300 python tools/time_two_pass.py
timeout 300 python tools/micro/stream_ceiling.py
} > gpurun_out/sweep1.txt 2>&1
