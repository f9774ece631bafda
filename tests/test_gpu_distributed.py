"""Multi-rank slab decomposition ON THE GPU (SlabSolver: interior/boundary launches of the fused
kernel with periodic_z = 0 and ghost planes), 2 and 3 ranks sharing one B200 over gloo (the halo
planes are staged through the host; production runs exchange them with NCCL over NVLink).
The gathered field must equal the single-field run bit for bit."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, order_n, cells, steps, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1609_09841_b200 as hb
        from paper_1609_09841_b200.distributed import SlabSolver, slab_bounds
        torch.cuda.set_device(0)
        cfg = hb.StepConfig(variant="separable")
        solver = SlabSolver(cells, order_n, cfg)
        solver.init(hb.plane_wave())
        for _ in range(steps):
            solver.step()
        solver.check()
        local = solver.state.cpu()
        m1, m2, m3 = cells
        if rank == 0:
            parts = [local]
            for r in range(1, world):
                z0, z1 = slab_bounds(m3, world, r)
                t = torch.empty((z1 - z0,) + tuple(local.shape[1:]), dtype=torch.float64)
                dist.recv(t, src=r)
                parts.append(t)
            got = torch.cat(parts)
            grid = hb.GridSpec(cells)
            state = hb.init_field(hb.plane_wave(), grid, order_n)
            scratch = hb.DofField.zeros(grid.with_parity("dual"), order_n)
            ops = hb.OperatorSet.for_grid(grid, order_n)
            for _ in range(steps):
                hb.full_step(state, scratch, cfg, ops, dt=solver.dt)
            with open(result_path, "w") as fh:
                fh.write("ok" if torch.equal(got, state.tensor.cpu()) else "mismatch")
        else:
            dist.send(local.contiguous(), dst=0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,order_n,cells", [(2, 3, (16, 14, 12)), (3, 3, (9, 8, 10)), (2, 5, (8, 8, 6)),
                                                 (2, 1, (10, 9, 7))])
def test_slab_solver_multi_rank_on_gpu(world, order_n, cells, tmp_path):
    out = tmp_path / "result.txt"
    mp.start_processes(_worker, args=(world, _free_port(), order_n, cells, 3, str(out)), nprocs=world,
                       join=True, start_method="spawn")
    assert out.read_text() == "ok"
