# A/B of the current library against paper_1609_09841_b200/libh3b200_old.so (512^3 m=3 fused)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_1609_09841_b200/libh3b200.so
cp $L /tmp/new.so
{
timeout 900 python -m pytest tests -q -x -m gpu -k "separable or degenerate or slab or instab or fused or fullsize or shift" 2>&1 | tail -1
for r in 1 2 3; do
  cp paper_1609_09841_b200/libh3b200_old.so $L; echo -n "old "; timeout 200 python tools/time_fused.py 3 512 fused 10
  cp /tmp/new.so $L; echo -n "new "; timeout 200 python tools/time_fused.py 3 512 fused 10
done
} > gpurun_out/ab2.txt 2>&1
