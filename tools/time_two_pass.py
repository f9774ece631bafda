"""Time the two-kernel (two_pass) half step per kernel with CUDA events (package timings)."""
import sys
import torch
sys.path.insert(0, ".")
import _lib  # noqa: E402
_lib.select_library()
import paper_1609_09841_b200 as hb

for n, m in [(3, 128), (3, 256), (1, 256), (5, 128)]:
    grid = hb.GridSpec((m, m, m))
    cfg = hb.StepConfig(mode="two_pass", variant="separable")
    ops = hb.OperatorSet.for_grid(grid, n)
    st = hb.init_field(hb.plane_wave(), grid, n)
    sc = hb.DofField.empty(grid.with_parity("dual"), n)
    hb.full_step(st, sc, cfg, ops)
    t = {}
    for _ in range(3):
        hb.full_step(st, sc, cfg, ops, timings=t)
    nodes = m ** 3
    rec = t["reconstruction"] / 6
    evo = t["evolution"] / 6
    bytes_rec = nodes * 8 * ((n + 1) ** 3 + (2 * n + 2) ** 3)
    print(f"N={n} M={m}: recon {rec*1e3:.2f} ms ({bytes_rec/rec/1e9:.0f} GB/s)  "
          f"evolve {evo*1e3:.2f} ms ({bytes_rec/evo/1e9:.0f} GB/s)", flush=True)
    del st, sc
    torch.cuda.empty_cache()
