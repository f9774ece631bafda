"""Per-instruction shared-memory excess wavefronts from an ncu source-page CSV (SASS view)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ie = hdr.index("L1 Wavefronts Shared Excessive")
iw = hdr.index("L1 Wavefronts Shared")
ii = hdr.index("L1 Wavefronts Shared Ideal")
tot = sum(float(r[ie] or 0) for r in data) or 1
print(f"total excessive {tot:.3e}, total {sum(float(r[iw] or 0) for r in data):.3e}")
for i, r in enumerate(data):
    e = float(r[ie] or 0)
    if e > 0.02 * tot:
        print(f"{i:5d} {100 * e / tot:5.1f}% of excess  wf {float(r[iw]):.2e} ideal {float(r[ii] or 0):.2e}  {r[1].strip()[:70]}")
