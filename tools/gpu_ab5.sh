# A/B of the current library against paper_1609_09841_b200/libh3b200_old.so (m=5 256^3 fused and two-pass)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_1609_09841_b200/libh3b200.so
cp $L /tmp/new.so
{
timeout 900 python -m pytest tests -q -x -m gpu -k "separable or fused or two_pass or recon or degenerate" 2>&1 | tail -1
for r in 1 2; do
  for mode in two_pass; do
    cp paper_1609_09841_b200/libh3b200_old.so $L; echo -n "old "; timeout 300 python tools/time_fused.py 5 256 $mode 4
    cp /tmp/new.so $L; echo -n "new "; timeout 300 python tools/time_fused.py 5 256 $mode 4
  done
done
} > gpurun_out/ab5.txt 2>&1
