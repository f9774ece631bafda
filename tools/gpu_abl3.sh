# literal kernel variants: base vs in-place w vs in-place + 3 CTAs/SM (N=3, 256^3 and N=5 128^3)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_1609_09841_b200/libh3b200.so
cp $L /tmp/cur.so
{
for v in base inp lb3 base inp lb3; do
  cp paper_1609_09841_b200/libh3b200_$v.so $L
  echo "== $v"; timeout 300 python tools/time_literal.py 3 256 2>&1 | grep literal
done
cp paper_1609_09841_b200/libh3b200_lb3.so $L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "literal or golden" 2>&1 | tail -1
} > gpurun_out/abl3.txt 2>&1
cp /tmp/cur.so $L
