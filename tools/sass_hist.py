"""Per-kernel SASS instruction histogram of libh3b200.so (static counts, cuobjdump -sass):
the evidence that the hot kernels run on the FP64 tensor cores (DMMA.8x8x4), stage tiles with
bulk async copies (UBLKCP) tracked by mbarriers (SYNCS), and how many shared-memory and global
instructions each carries.

usage: python tools/sass_hist.py [LIB] > profiles/r02_sass_histogram.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_1609_09841_b200" / "libh3b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
demangle = lambda names: subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,  # noqa: E731
                                        text=True).stdout.splitlines()

KEYS = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG", "BAR", "SHFL",
        "HMMA", "UTCMMA", "UTMALDG"]
kernels = []
cur, counts = None, None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        if cur:
            kernels.append((cur, counts))
        cur, counts = m.group(1), collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        op = m.group(1)
        counts["total"] += 1
        counts[op] += 1
if cur:
    kernels.append((cur, counts))
names = demangle([k for k, _ in kernels])
hot = re.compile(r"sep_fused|recon_dmma|sep_evolve|dmma_cp|literal_kernel<double, 3|recon_sep|h3::cell")
print(f"# static SASS histogram of {Path(lib).name} (cuobjdump -sass; sm_100a)")
print(f"# opcode families counted by prefix: {', '.join(KEYS)}")
for (mangled, c), name in zip(kernels, names):
    if not hot.search(name):
        continue
    fam = collections.Counter()
    for op, v in c.items():
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                fam[k] += v
    exact = {op: v for op, v in c.items() if op.startswith(("DMMA", "UBLKCP", "SYNCS"))}
    print(f"\n{name[:160]}")
    print(f"  total {c['total']}  " + "  ".join(f"{k} {fam[k]}" for k in KEYS if fam[k]))
    print("  exact: " + ", ".join(f"{k} {v}" for k, v in sorted(exact.items())))
