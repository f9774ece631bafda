"""HostStepper (host-resident field) throughput vs chunk size, and raw PCIe copy rates."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_09841_b200 as hb  # noqa: E402

n, m = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 512
grid = hb.GridSpec((m, m, m))
cfg = hb.StepConfig(variant="separable")
st = hb.init_field(hb.plane_wave(), grid, n)
host = torch.empty(st.tensor.shape, dtype=torch.float64, pin_memory=True)
host.copy_(st.tensor)
del st
torch.cuda.empty_cache()
dev = torch.empty(host.numel() // 16, dtype=torch.float64, device="cuda")
hv = host.view(-1)[: dev.numel()]
nbytes = dev.numel() * 8
for name, fn in (("H2D", lambda: dev.copy_(hv, non_blocking=True)), ("D2H", lambda: hv.copy_(dev, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(f"{name} {nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dev2 = torch.empty_like(dev)
hv2 = host.view(-1)[dev.numel(): 2 * dev.numel()]
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    dev.copy_(hv, non_blocking=True)
with torch.cuda.stream(s2):
    hv2.copy_(dev2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D+D2H concurrent {2 * nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s total", flush=True)
del dev, dev2
torch.cuda.empty_cache()
plane = m * m * (n + 1) ** 3 * 8
for arg in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8", "16", "32", "64"]):
    planes, ramp = int(arg.rstrip("r")), arg.endswith("r")  # "16r": ramped chunk sizes
    stp = hb.HostStepper(host, grid, n, cfg, chunk_planes=planes, ramp=ramp)
    stp.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(2):
        stp.step(step_index=k)
    dt = (time.perf_counter() - t0) / 2
    print(f"chunk {planes}{'r' if ramp else ''} planes ({planes * plane / 1e9:.1f} GB, {len(stp.chunks)} chunks): {dt:.3f} s/step, "
          f"{m ** 3 * (n + 1) ** 3 / dt:.3e} DOF-updates/s, {(stp.h2d_bytes + stp.d2h_bytes) / dt / 1e9:.1f} GB/s PCIe", flush=True)
    del stp
    torch.cuda.empty_cache()
