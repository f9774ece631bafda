cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -q -x -m gpu -k "separable or degenerate or convergence or fused" 2>&1 | tail -1
timeout 200 python tools/time_fused.py 5 256 fused 4
timeout 200 python tools/time_fused.py 5 256 fused 4
} > gpurun_out/n5l.txt 2>&1
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum -k regex:dmma_cp -s 2 -c 1 python tools/time_fused.py 5 128 fused 1 >> gpurun_out/n5l.txt 2>&1
