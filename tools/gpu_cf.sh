cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
H3_DMMA_CFG=30 timeout 900 python -m pytest tests -q -x -m gpu -k "separable or degenerate or slab or instab or fused or fullsize or shift" 2>&1 | tail -1
for c in 0 30 0 30; do H3_DMMA_CFG=$c timeout 200 python tools/time_fused.py 3 512 fused 6; done
} > gpurun_out/cf.txt 2>&1
for c in 0 30; do H3_DMMA_CFG=$c timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum -k regex:sep_fused -s 2 -c 1 python tools/time_fused.py 3 256 fused 1 >> gpurun_out/cf.txt 2>&1; done
