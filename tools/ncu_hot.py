"""Summarise an `ncu --page source --csv --print-source sass` dump: hottest SASS lines with stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
tot = sum(int(r[si]) for r in data) or 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
for i, r in enumerate(data):
    s = int(r[si])
    if s > tot * thr:
        top = sorted(((int(r[j]) if r[j] else 0, reasons[k][6:]) for k, j in enumerate(ri)), reverse=True)[:3]
        print(f"{i:5d} {100 * s / tot:5.1f}% {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in top if v))
