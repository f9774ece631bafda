cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2l_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest_gpu.log
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --kernel-name regex:dmma_ws python tools/sanitize.py > gpurun_out/r2l_san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/r2l_san_$tool.txt; done
timeout 900 python bench.py --no-cpu > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "rc=$?" >> gpurun_out/r2l_bench.err
echo done
