cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "recon or ring or two_pass or separable" 2>&1 | tail -5
timeout 300 python tools/time_two_pass.py
H3_RECON_IMPL=sep timeout 300 python tools/time_two_pass.py
timeout 300 python tools/time_fused.py 5 256 two_pass 2
} > gpurun_out/recon1.txt 2>&1
