"""Convert the ncu launch list (--metrics gpu__time_duration.sum --csv --log-file) to profiles JSON.

usage: python tools/launches_json.py gpurun_out/launches.csv profiles/r01_bench_launches.json
"""
import csv
import json
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
launches = [{"id": r[0], "kernel": r[ki][:140], "ms": float(r[vi].replace(",", "")) * scale[r[ui]]}
            for r in data if r[mi] == "gpu__time_duration.sum"]
json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 "
                      "--warmup 1 --no-e2e --no-cpu --no-extras",
           "note": "cold-cache serialised launches; includes the untimed device init of the field; every timed "
                   "launch is the fused half-step kernel",
           "launches": launches}, open(sys.argv[2], "w"), indent=1)
print(len(launches), "launches")
