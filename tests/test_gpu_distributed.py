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


def _worker(rank, world, port, order_n, cells, steps, result_path, halo, mode="fused"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1609_09841_b200 as hb
        from paper_1609_09841_b200.distributed import SlabSolver, slab_bounds
        torch.cuda.set_device(0)
        cfg = hb.StepConfig(mode=mode, variant="separable", coeff_budget_bytes=mode == "two_pass" and 3 * 10**6 or None)
        solver = SlabSolver(cells, order_n, cfg, halo=halo)
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
            want_halo = {"auto": "p2p" if order_n in (3, 5) and mode == "fused" else "nccl"}.get(halo, halo)
            with open(result_path, "w") as fh:
                fh.write("ok" if torch.equal(got, state.tensor.cpu()) and solver.halo == want_halo else
                         f"mismatch (halo {solver.halo}: {solver.halo_note})")
        else:
            dist.send(local.contiguous(), dst=0)
        dist.barrier()  # peers keep their buffers mapped until everyone is done
        solver.close()
    finally:
        dist.destroy_process_group()





@pytest.mark.parametrize("world,order_n,cells,halo", [(2, 3, (16, 14, 12), "nccl"), (3, 3, (9, 8, 10), "nccl"),
                                                      (2, 5, (8, 8, 6), "nccl"), (2, 1, (10, 9, 7), "nccl"),
                                                      (2, 3, (16, 14, 12), "p2p"), (3, 3, (9, 8, 10), "p2p"),
                                                      (2, 5, (8, 8, 6), "p2p"), (2, 3, (16, 14, 12), "auto"),
                                                      (2, 1, (10, 9, 7), "auto")])
def test_slab_solver_multi_rank_on_gpu(world, order_n, cells, halo, tmp_path):
    """halo="nccl": ghost planes copied by the exchange (staged through gloo here); halo="p2p": the
    kernel reads the neighbour's plane in place through a CUDA-IPC mapping (here: processes
    sharing one GPU, so the mapping is same-device)."""
    out = tmp_path / "result.txt"
    mp.start_processes(_worker, args=(world, _free_port(), order_n, cells, 3, str(out), halo), nprocs=world,
                       join=True, start_method="spawn")
    assert out.read_text() == "ok"


@pytest.mark.parametrize("world,order_n,cells,halo", [(2, 3, (16, 14, 12), "auto"), (3, 5, (8, 8, 9), "nccl"),
                                                      (2, 1, (10, 9, 7), "nccl")])
def test_slab_solver_two_kernel_multi_rank_on_gpu(world, order_n, cells, halo, tmp_path):
    """The two-kernel step on slabs (recon_pass reading the NCCL ghost plane with periodic_z = 0,
    then evolve_pass, in small coefficient chunks so a slab spans several): bit-identical to the
    single-field two-kernel run; halo="auto" resolves to the NCCL copy for this mode."""
    out = tmp_path / "result.txt"
    mp.start_processes(_worker, args=(world, _free_port(), order_n, cells, 3, str(out), halo, "two_pass"),
                       nprocs=world, join=True, start_method="spawn")
    assert out.read_text() == "ok"


@pytest.mark.parametrize("order_n,cells", [(3, (16, 14, 12)), (5, (8, 8, 6))])
def test_slab_solver_p2p_single_rank(order_n, cells):
    """One rank: the p2p halo maps the rank's own boundary planes (periodic wrap) -- the
    ghost-pointer kernel path against the periodic single-field run, bit for bit."""
    import paper_1609_09841_b200 as hb
    from paper_1609_09841_b200.distributed import SlabSolver
    cfg = hb.StepConfig(variant="separable")
    solver = SlabSolver(cells, order_n, cfg, halo="p2p")
    solver.init(hb.plane_wave())
    grid = hb.GridSpec(cells)
    state = hb.init_field(hb.plane_wave(), grid, order_n)
    scratch = hb.DofField.zeros(grid.with_parity("dual"), order_n)
    ops = hb.OperatorSet.for_grid(grid, order_n)
    for _ in range(3):
        solver.step()
        hb.full_step(state, scratch, cfg, ops, dt=solver.dt)
    solver.check()
    assert torch.equal(solver.state, state.tensor)


def _bad_worker(rank, world, port, cells, bad, halo, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1609_09841_b200 as hb
        from paper_1609_09841_b200.distributed import SlabSolver
        torch.cuda.set_device(0)
        cfg = hb.StepConfig(variant="separable")
        solver = SlabSolver(cells, 3, cfg, halo=halo)
        solver.init(hb.plane_wave())
        if solver.z0 <= bad[0] < solver.z1:
            solver.state[(bad[0] - solver.z0,) + tuple(bad[1:])] = float("inf")
        before = solver.state.clone()
        err = None
        try:
            solver.step()
            solver.check(step_index=4)
        except hb.InstabilityError as e:
            err = (e.node, e.step)
        # the reference raises after the first half step with the state untouched: the second
        # half step is skipped on EVERY rank (collective guard), and so is any later step
        untouched = torch.equal(solver.state, before)
        solver.step()
        untouched = untouched and torch.equal(solver.state, before)
        errs = [None] * world
        dist.all_gather_object(errs, (err, untouched))
        if rank == 0:
            grid = hb.GridSpec(cells)
            state = hb.init_field(hb.plane_wave(), grid, 3)
            state.tensor[bad] = float("inf")
            scratch = hb.DofField.zeros(grid.with_parity("dual"), 3)
            with pytest.raises(hb.InstabilityError) as ref:
                hb.full_step(state, scratch, cfg, hb.OperatorSet.for_grid(grid, 3), dt=solver.dt, step_index=4)
            want = (ref.value.node, ref.value.step)
            with open(result_path, "w") as fh:
                fh.write("ok" if all(e == (want, True) for e in errs) else f"mismatch {errs} vs {want}")
        dist.barrier()
        solver.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_slab_solver_instability_is_collective(halo, tmp_path):
    """A non-finite value on one rank makes EVERY rank raise the same InstabilityError (the
    first bad node of the whole grid, as full_step reports it), so no rank is left waiting in
    the next halo exchange."""
    out = tmp_path / "result.txt"
    mp.start_processes(_bad_worker, args=(2, _free_port(), (8, 7, 8), (5, 2, 3, 0, 0, 0), halo, str(out)),
                       nprocs=2, join=True, start_method="spawn")
    assert out.read_text() == "ok"


def _fail_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1609_09841_b200 as hb
        from paper_1609_09841_b200 import _native
        from paper_1609_09841_b200.distributed import SlabSolver
        torch.cuda.set_device(0)
        if rank == 1:  # this rank cannot export its buffers (e.g. no IPC support)
            _native.lib().h3_ipc_export = lambda *args: -1
        cells = (16, 14, 12)
        cfg = hb.StepConfig(variant="separable")
        solver = SlabSolver(cells, 3, cfg, halo="auto")
        solver.init(hb.plane_wave())
        for _ in range(2):
            solver.step()
        solver.check()
        halos = [None] * world
        dist.all_gather_object(halos, (solver.halo, solver.halo_note))
        states = [None] * world
        dist.all_gather_object(states, solver.state.cpu())
        if rank == 0:
            grid = hb.GridSpec(cells)
            state = hb.init_field(hb.plane_wave(), grid, 3)
            scratch = hb.DofField.zeros(grid.with_parity("dual"), 3)
            for _ in range(2):
                hb.full_step(state, scratch, cfg, hb.OperatorSet.for_grid(grid, 3), dt=solver.dt)
            ok = all(h == "nccl" and "p2p setup failed" in note for h, note in halos) \
                and torch.equal(torch.cat(states), state.tensor.cpu())
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else f"mismatch {halos}")
        dist.barrier()
        solver.close()
    finally:
        dist.destroy_process_group()


def test_slab_solver_p2p_setup_failure_on_one_rank_falls_back_everywhere(tmp_path):
    """halo="auto": when one rank cannot set up the IPC mapping, every rank agrees on the NCCL
    halo (no rank waits in a collective the others skipped) and the result is unchanged."""
    out = tmp_path / "result.txt"
    mp.start_processes(_fail_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    assert out.read_text() == "ok"
