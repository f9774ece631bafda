cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in 11 12; do H3_LIB=build/libh3b200_measure.so H3_DMMA5_CFG=$c timeout 300 python tools/variant_check.py 5 40 36 20; done > gpurun_out/r2d_check.txt 2>&1
tools/ab.sh 2 "base:" "L2:H3_DMMA5_CFG=9" "Vonly:H3_DMMA5_CFG=11" "Wonly:H3_DMMA5_CFG=12" -- tools/time_fused.py 5 256 fused 4 > gpurun_out/r2d_ab5.txt 2>&1
tools/ab.sh 2 "c12:" "c22:H3_DMMA_CLUSTER_X=2" "c21:H3_DMMA_CLUSTER_X=2 H3_DMMA_CLUSTER_Y=1" "c11:H3_DMMA_CLUSTER_Y=1" "c14:H3_DMMA_CLUSTER_Y=4" -- tools/energy.py 512 40 > gpurun_out/r2d_cluster.txt 2>&1
echo done
