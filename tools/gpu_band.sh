cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA_BAND=16 timeout 900 python -m pytest tests -q -x -m gpu -k "separable or degenerate or slab or instab or fused" 2>&1 | tail -1
for b in 0 8 16 32 0 16; do H3_DMMA_BAND=$b timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/band.txt 2>&1
H3_DMMA_BAND=16 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sep_fused -s 2 -c 1 python tools/time_fused.py 3 512 fused 1 >> gpurun_out/band.txt 2>&1
