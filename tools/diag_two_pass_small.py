"""Host-side cost breakdown of a small two-pass half step (diagnostic)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1609_09841_b200 as hb  # noqa: E402
from paper_1609_09841_b200 import _native, pipeline  # noqa: E402

grid = hb.GridSpec((16, 16, 16))
n = 3
cfg = hb.StepConfig(mode="two_pass")
ops = hb.OperatorSet.for_grid(grid, n)
st = hb.init_field(hb.plane_wave(), grid, n)
sc = hb.DofField.zeros(grid.with_parity("dual"), n)
for _ in range(3):
    hb.full_step(st, sc, cfg, ops)
torch.cuda.synchronize()


def tm(label, fn, k=50):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host {1e6 * (t1 - t0) / k:.1f} us/call, incl. drain {1e6 * (t2 - t0) / k:.1f}", flush=True)


tm("mem_get_info", lambda: torch.cuda.mem_get_info())
tm("coeff_chunk_planes", lambda: pipeline._coeff_chunk_planes(grid, n, 8, None))
tm("torch.empty 16x16x16x512", lambda: torch.empty((16, 16, 16, 8, 8, 8), dtype=torch.float64, device="cuda"))
dt = hb.select_dt(grid, cfg)
fa = pipeline._factor_arrays(ops, np.float64, dt / 2, 21)
tm("factor_arrays", lambda: pipeline._factor_arrays(ops, np.float64, dt / 2, 21))
coeff = torch.empty((16, 16, 16, 8, 8, 8), dtype=torch.float64, device="cuda")
lib = _native.lib()
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = pipeline._ptr
tm("h3_recon_pass", lambda: lib.h3_recon_pass(ctypes.c_void_p(st.tensor.data_ptr()), ctypes.c_void_p(coeff.data_ptr()),
                                              16, 16, 16, n, P(fa[0]), 0, 0, 16, 1, 0, sh, None))
tm("h3_evolve_pass", lambda: lib.h3_evolve_pass(ctypes.c_void_p(coeff.data_ptr()), ctypes.c_void_p(sc.tensor.data_ptr()),
                                                16, 16, 16, n, P(fa[1]), P(fa[2]), P(fa[3]), P(fa[4]), 21, 0, 16, 0,
                                                sh, None, None))
tm("h3_fused_pass", lambda: lib.h3_fused_pass(ctypes.c_void_p(st.tensor.data_ptr()), ctypes.c_void_p(sc.tensor.data_ptr()),
                                              16, 16, 16, n, P(fa[0]), P(fa[1]), P(fa[2]), P(fa[3]), P(fa[4]), 21, 0, 0,
                                              16, 1, 0, sh, None, None))
tm("half_step two_pass", lambda: hb.half_step(st, sc, cfg, ops, _check=False))
tm("half_step fused", lambda: hb.half_step(st, sc, hb.StepConfig(), ops, _check=False))
