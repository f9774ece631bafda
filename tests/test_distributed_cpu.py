"""Multi-process CPU tests (gloo, world_size 2 and 3) of the slab decomposition.

The B200 path exchanges one ghost plane per half step with NCCL send/recv and runs
the half-step kernel on each slab with periodic_z = 0
(paper_1609_09841_b200/distributed.py).  Here the same exchange code runs over
gloo on CPU tensors and the per-slab compute is the CPU oracle on the
(L + 2)-plane slab buffer (test infrastructure); the gathered result must equal
the single-process oracle run bit for bit, for both gather offsets.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import refmodel as rm
from paper_1609_09841_b200.distributed import exchange_halo, halo_plan, slab_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_slab_bounds_partition():
    for m3 in (7, 8, 64, 513):
        for world in (1, 2, 3, 4, 8):
            if m3 < world:
                continue
            spans = [slab_bounds(m3, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m3
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_halo_plan_directions():
    # off = 0 reads nodes c, c+1: ghost_hi <- first plane of rank+1, send first plane to rank-1
    assert halo_plan(0, 1, 4, 10) == (1, 0, 11, 2)
    # off = -1 reads nodes c-1, c: ghost_lo <- last plane of rank-1, send last plane to rank+1
    assert halo_plan(-1, 1, 4, 10) == (10, 2, 0, 0)
    assert halo_plan(0, 0, 4, 10)[1] == 3 and halo_plan(-1, 3, 4, 10)[1] == 0  # periodic ring
    with pytest.raises(ValueError):
        halo_plan(1, 0, 2, 4)


def _worker(rank, world, port, order_n, cells, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m1, m2, m3 = cells
        n = order_n + 1
        z0, z1 = slab_bounds(m3, world, rank)
        full = rm.init_field(rm.plane_wave_terms(), cells, (1.0, 1.0, 1.0), order_n)
        L = z1 - z0
        state = torch.zeros((L + 2, m2, m1, n, n, n), dtype=torch.float64)
        scratch = torch.zeros_like(state)
        state[1:-1] = torch.from_numpy(full[z0:z1])
        dt = rm.select_dt(cells)
        h_mat, f1, f2, f3, cf = rm.factor_arrays(order_n, cells, (1.0, 1.0, 1.0), dt / 2, rm.default_stages(order_n))
        for _ in range(steps):
            for src, dst, off in ((state, scratch, 0), (scratch, state, -1)):
                exchange_halo(src, off)
                out = np.zeros((L + 2, m2, m1, n, n, n))
                # buffer cells 1..L of a periodic oracle pass over the slab buffer never wrap
                rm.fused_pass(np.ascontiguousarray(src.numpy()), out, h_mat, f1, f2, f3, cf, off)
                dst[1:-1] = torch.from_numpy(out[1:-1])
        gathered = [torch.zeros((b - a, m2, m1, n, n, n), dtype=torch.float64)
                    for a, b in (slab_bounds(m3, world, r) for r in range(world))]
        if rank == 0:
            gathered[0].copy_(state[1:-1])
            for r in range(1, world):
                dist.recv(gathered[r], src=r)  # slabs may differ in size: plain point-to-point
            got = torch.cat(gathered).numpy()
            ref = full.copy()
            sc = np.zeros_like(ref)
            for _ in range(steps):
                rm.full_step(ref, sc, order_n, cells, (1.0, 1.0, 1.0), dt)
            assert np.array_equal(got, ref), "slab-decomposed run differs from the single-field run"
        else:
            dist.send(state[1:-1].contiguous(), dst=0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cells,order_n", [(2, (6, 5, 8), 1), (3, (4, 5, 7), 2), (2, (5, 4, 6), 3)])
def test_slab_halo_exchange_matches_single_field(world, cells, order_n):
    mp.start_processes(_worker, args=(world, _free_port(), order_n, cells, 3, None), nprocs=world,
                       join=True, start_method="spawn")


def _agree_worker(rank, world, port, per_rank, want):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_09841_b200.distributed import agree_first_bad
        got = agree_first_bad(per_rank[rank])
        assert got == want, (rank, got, want)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("per_rank,want", [([[-1, 7], [12, -1]], [12, 7]), ([[-1, -1], [-1, -1]], [-1, -1]),
                                           ([[30, 9], [4, 11]], [4, 9])])
def test_instability_agreement_is_min_over_ranks(per_rank, want):
    """Every rank gets the first bad global node per half step (min over ranks, -1 = none)."""
    mp.start_processes(_agree_worker, args=(2, _free_port(), per_rank, want), nprocs=2, join=True,
                       start_method="spawn")
