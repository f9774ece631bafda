cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/abl_clocks.csv &
SMI=$!
{
for c in 6 11 14 15 16 6; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/abl.txt 2>&1
kill $SMI
