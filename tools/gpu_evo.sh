cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "two_pass or separable or recon or shift or linearity" 2>&1 | tail -1
timeout 300 python tools/time_two_pass.py 2>&1
} > gpurun_out/evo.txt 2>&1
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum -k regex:sep_evolve -s 2 -c 1 python tools/time_fused.py 3 128 two_pass 1 >> gpurun_out/evo.txt 2>&1
