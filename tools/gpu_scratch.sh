cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_ws.py > gpurun_out/r2o_race.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_ws.py 17 9 31 > gpurun_out/r2o_sync.txt 2>&1
for c in 45; do H3_LIB=build/libh3b200_measure.so H3_DMMA5_CFG=$c timeout 90 python tools/variant_check.py 5 40 36 20; done > gpurun_out/r2o_check.txt 2>&1
tools/ab.sh 3 "ws:" "lockstep:H3_DMMA5_CFG=13" -- tools/time_fused.py 5 256 fused 4 > gpurun_out/r2o_ab5.txt 2>&1
echo done
