cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "configs or full or fused_vs_two_pass" -q -rP > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
tools/ab.sh 2 "base:" "c3ilp:H3_DMMA5_CFG=3" "c4st2:H3_DMMA5_CFG=4" "c5_2x8:H3_DMMA5_CFG=5" "c6_2x8ilp:H3_DMMA5_CFG=6" "c7_3x6:H3_DMMA5_CFG=7" "c8_4x5:H3_DMMA5_CFG=8" -- tools/time_fused.py 5 256 fused 4 > gpurun_out/r2b_ab5.txt 2>&1
echo done
