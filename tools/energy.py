"""Energy per half step of the N=3 fused kernel (NVML total-energy counter), for the kernel
variant selected by H3_DMMA_CFG (ablations: 11 no stores, 14 DMMA -> register update, 15 both,
16 the same structure with all work), plus a device-to-device copy of the same bytes and the
idle draw.  Prints J per half step, mean W and the SM clock under load.

usage: H3_DMMA_CFG=16 python tools/energy.py [CELLS] [HALF_STEPS] [copy|idle|kernel] [ORDER]
"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 60
what = sys.argv[3] if len(sys.argv) > 3 else "kernel"
order = int(sys.argv[4]) if len(sys.argv) > 4 else 3
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
clocks = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.05)


grid = hb.GridSpec((m, m, m))
cfg = hb.StepConfig(variant="separable")
if what == "kernel":
    ops = hb.OperatorSet.for_grid(grid, order)
    a = hb.init_field(hb.plane_wave(), grid, order)
    b = hb.DofField.empty(grid.with_parity("dual"), order)
    dt = hb.select_dt(grid, cfg)
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")

    def one(i):
        src, dst = (a, b) if i % 2 == 0 else (b, a)
        hb.half_step(src, dst, cfg, ops, dt=dt, _flag=flag, _check=False)
elif what == "copy":
    x = torch.empty((m, m, m) + (order + 1,) * 3, dtype=torch.float64, device="cuda").uniform_()
    y = torch.empty_like(x)

    def one(i):
        (y if i % 2 == 0 else x).copy_(x if i % 2 == 0 else y)
else:
    def one(i):
        time.sleep(0.05)

for i in range(6):
    one(i)
torch.cuda.synchronize()
th = threading.Thread(target=sample)
th.start()
e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
t0 = time.perf_counter()
for i in range(k):
    one(i)
torch.cuda.synchronize()
t1 = time.perf_counter()
e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
stop.set()
th.join()
joules = (e1 - e0) / 1e3
clk = sorted(clocks)[len(clocks) // 2] if clocks else 0
print(f"{what:6s} N={order} cfg={os.environ.get('H3_DMMA_CFG', '0'):3s} {1e3 * (t1 - t0) / k:8.3f} ms/half-step  "
      f"{joules / k:7.2f} J/half-step  {joules / (t1 - t0):6.0f} W  sm {clk} MHz")
