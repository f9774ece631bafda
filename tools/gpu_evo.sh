cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
for c in 8 1 2; do echo "CPB=$c"; H3_EVOLVE_CPB=$c timeout 300 python tools/time_two_pass.py 2>&1 | head -2; done
} > gpurun_out/evo.txt 2>&1
