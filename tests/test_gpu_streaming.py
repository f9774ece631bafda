"""Host-resident stepping (streaming.HostStepper) against the device-resident full_step:
bit-identical states, including one-chunk, two-chunk and ragged chunkings, and the same
InstabilityError (node, step) as the reference's raise-after-half-step semantics."""

import numpy as np
import pytest
import torch

import paper_1609_09841_b200 as hb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order_n,cells,chunk", [(3, (12, 10, 9), 4), (3, (8, 8, 8), 8), (1, (9, 7, 6), 3),
                                                  (5, (6, 5, 7), 2), (3, (10, 9, 11), 5), (2, (7, 6, 5), 100)])
def test_host_stepper_bitwise_equals_full_step(order_n, cells, chunk):
    grid = hb.GridSpec(cells)
    cfg = hb.StepConfig(variant="separable")
    ops = hb.OperatorSet.for_grid(grid, order_n)
    state = hb.init_field(hb.plane_wave(), grid, order_n)
    scratch = hb.DofField.zeros(grid.with_parity("dual"), order_n)
    host = torch.empty(state.tensor.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(state.tensor)
    stepper = hb.HostStepper(host, grid, order_n, cfg, chunk_planes=chunk)
    dt = hb.select_dt(grid, cfg)
    for k in range(3):
        hb.full_step(state, scratch, cfg, ops, dt=dt, step_index=k)
        stepper.step(dt=dt, step_index=k)
    assert torch.equal(host, state.tensor.cpu())


def test_host_stepper_pageable_host_memory():
    grid = hb.GridSpec((8, 6, 6))
    cfg = hb.StepConfig(variant="separable")
    state = hb.init_field(hb.plane_wave(), grid, 3)
    scratch = hb.DofField.zeros(grid.with_parity("dual"), 3)
    host = state.tensor.cpu().clone()
    hb.HostStepper(host, grid, 3, cfg, chunk_planes=2).step()
    hb.full_step(state, scratch, cfg, hb.OperatorSet.for_grid(grid, 3))
    assert torch.equal(host, state.tensor.cpu())


def test_host_stepper_reports_instability_like_full_step():
    grid = hb.GridSpec((8, 7, 6))
    cfg = hb.StepConfig(variant="separable")
    ops = hb.OperatorSet.for_grid(grid, 3)
    state = hb.init_field(hb.plane_wave(), grid, 3)
    t = state.tensor
    t[4, 3, 2, 0, 0, 0] = float("inf")
    t[5, 1, 6, 1, 0, 0] = float("nan")
    host = t.cpu().clone()
    scratch = hb.DofField.zeros(grid.with_parity("dual"), 3)
    with pytest.raises(hb.InstabilityError) as ref:
        hb.full_step(state, scratch, cfg, ops, step_index=7)
    with pytest.raises(hb.InstabilityError) as got:
        hb.HostStepper(host, grid, 3, cfg, chunk_planes=2).step(step_index=7)
    assert got.value.node == ref.value.node and got.value.step == ref.value.step


def test_host_stepper_validates_arguments():
    grid = hb.GridSpec((4, 4, 4))
    with pytest.raises(ValueError):
        hb.HostStepper(torch.zeros((4, 4, 4, 2, 2, 2)), grid, 3)  # wrong shape for N=3
    with pytest.raises(ValueError):
        hb.HostStepper(torch.zeros((4, 4, 4, 4, 4, 4)), grid, 3, hb.StepConfig(mode="two_pass"))


def _slab_worker(rank, world, port, order_n, cells, chunk, steps, result_path, bad):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_09841_b200.distributed import slab_bounds
        torch.cuda.set_device(0)
        grid = hb.GridSpec(cells)
        cfg = hb.StepConfig(variant="separable")
        full = hb.init_field(hb.plane_wave(), grid, order_n).tensor
        if bad is not None:
            full[bad] = float("inf")
        z0, z1 = slab_bounds(cells[2], world, rank)
        host = full[z0:z1].cpu().clone().pin_memory()
        stepper = hb.HostStepper(host, grid, order_n, cfg, chunk_planes=chunk)
        dt = hb.select_dt(grid, cfg)
        err = None
        try:
            for k in range(steps):
                stepper.step(dt=dt, step_index=k)
        except hb.InstabilityError as e:
            err = (e.node, e.step)
        parts = [None] * world
        dist.all_gather_object(parts, (host, err))
        if rank == 0:
            got = torch.cat([p[0] for p in parts])
            errs = [p[1] for p in parts if p[1] is not None]
            state = hb.init_field(hb.plane_wave(), grid, order_n)
            if bad is not None:
                state.tensor[bad] = float("inf")
            scratch = hb.DofField.zeros(grid.with_parity("dual"), order_n)
            ops = hb.OperatorSet.for_grid(grid, order_n)
            want_err = None
            try:
                for k in range(steps):
                    hb.full_step(state, scratch, cfg, ops, dt=dt, step_index=k)
            except hb.InstabilityError as e:
                want_err = (e.node, e.step)
            if want_err is not None:
                ok = want_err in errs
            else:
                ok = torch.equal(got, state.tensor.cpu()) and not errs
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else f"mismatch {errs} {want_err}")
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,order_n,cells,chunk,bad", [(2, 3, (10, 9, 12), 2, None), (3, 3, (8, 7, 10), 100, None),
                                                         (2, 1, (9, 7, 9), 3, None), (2, 5, (6, 5, 8), 2, None),
                                                         (2, 3, (8, 7, 8), 2, (6, 2, 3, 0, 0, 0))])
def test_host_stepper_slabs_multi_rank(world, order_n, cells, chunk, bad, tmp_path):
    """Each rank streams its own x3 slab from host memory, the wrap planes exchanged with the
    neighbour ranks (gloo here, processes sharing one GPU): the gathered field equals the
    single-field full_step bit for bit, and an instability is reported at the same node."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "result.txt"
    mp.start_processes(_slab_worker, args=(world, port, order_n, cells, chunk, 3, str(out), bad), nprocs=world,
                       join=True, start_method="spawn")
    assert out.read_text() == "ok"
