# energy per half step: fused kernel variants, a copy of the same bytes, idle
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 120 python tools/energy.py 512 40 idle
timeout 300 python tools/energy.py 512 60 copy
for c in 0 16 11 14 15 6; do H3_DMMA_CFG=$c timeout 300 python tools/energy.py 512 60; done
timeout 300 python tools/energy.py 512 60 copy
} > gpurun_out/energy.txt 2>&1
