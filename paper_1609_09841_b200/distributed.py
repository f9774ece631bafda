"""Slab decomposition of the periodic grid along x3 with a one-plane halo per half step.

The reference has no multi-process path; this module is
the B200 scaling layer of SURVEY.md 8(e).  x3 is the outermost index of the
DOF layout [m3][m2][m1][n3][n2][n1], so a node plane is one contiguous
M1*M2*(N+1)^3 block.

Each rank stores its L local planes between two ghost planes:
    buf[0] = ghost_lo, buf[1 .. L] = local planes, buf[L+1] = ghost_hi.
A half step needs ONE neighbour plane, and the direction alternates with
the gather offset (reference gridkernels.py:46, g = c + off + a):
    off =  0 (primary -> dual): cell c needs nodes c, c+1  -> ghost_hi = first
             local plane of rank+1 (send my first plane to rank-1);
    off = -1 (dual -> primary): cell c needs nodes c-1, c  -> ghost_lo = last
             local plane of rank-1 (send my last plane to rank+1).
The ranks form a periodic ring.  Two halo implementations:

* "nccl" (default): an NCCL send/recv pair (over NVLink/NVSwitch) copies the
  neighbour's plane into the ghost plane; it is issued before the interior
  cell planes are launched, so it overlaps with them, and the one boundary
  cell plane that reads the ghost is launched after the exchange completes
  (h3_fused_pass with periodic_z = 0).
* "p2p": no copy at all -- the neighbours' field buffers are mapped through
  CUDA IPC once, and the kernel's TMA plane loads read the neighbour's
  boundary plane in place over NVLink (h3_fused_pass_halo); a stream-ordered
  all-reduce of one element per half step is the only collective (it orders
  the neighbours' previous half step before the read and the overwrite).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .field import GridSpec
from .pipeline import InstabilityError, OperatorSet, StepConfig, _factor_arrays, _node_of, _ptr, select_dt

__all__ = ["slab_bounds", "halo_plan", "exchange_halo", "agree_first_bad", "SlabSolver"]


def slab_bounds(m3: int, world: int, rank: int) -> tuple[int, int]:
    """Planes [z0, z1) owned by `rank` (the first m3 % world ranks get one extra)."""
    base, extra = divmod(m3, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def halo_plan(off: int, rank: int, world: int, local_planes: int):
    """(send_buf_index, send_to, recv_buf_index, recv_from) for one half step."""
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    if off == 0:
        return 1, prv, local_planes + 1, nxt
    if off == -1:
        return local_planes, nxt, 0, prv
    raise ValueError(f"off must be 0 or -1, got {off}")


def exchange_halo(buf: torch.Tensor, off: int, group=None, async_op: bool = False):
    """Fill the ghost plane a half step with offset `off` reads (see module doc).

    `buf` has shape (L + 2, ...) with the ghost planes at both ends.  Works for
    CUDA tensors (NCCL) and CPU tensors (gloo).  Returns the list of pending
    works when async_op (empty when the exchange was a local copy).
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = buf.shape[0] - 2
    send_i, send_to, recv_i, recv_from = halo_plan(off, rank, world, local)
    if world == 1:
        buf[recv_i].copy_(buf[send_i])
        return []
    to_g = dist.get_global_rank(group, send_to) if group is not None else send_to
    from_g = dist.get_global_rank(group, recv_from) if group is not None else recv_from
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host tensors only: stage the planes (used to test the multi-rank GPU path
        # on one device; production runs use NCCL over NVLink)
        send, recv = buf[send_i].cpu(), torch.empty_like(buf[recv_i], device="cpu")
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, send, to_g, group),
                                         dist.P2POp(dist.irecv, recv, from_g, group)]):
            w.wait()
        buf[recv_i].copy_(recv)
        return []
    ops = [dist.P2POp(dist.isend, buf[send_i], to_g, group),
           dist.P2POp(dist.irecv, buf[recv_i], from_g, group)]
    works = dist.batch_isend_irecv(ops)
    if async_op:
        return works
    for w in works:
        w.wait()
    return []


def agree_first_bad(per_half: list[int], group=None, device=None) -> list[int]:
    """Make an instability report collective: `per_half` holds, for each half step in order,
    this rank's first non-finite node as a GLOBAL linear index ((m3 M2 + m2) M1 + m1, the
    reference's C-order scan) or -1; returns the minimum over all ranks per half step, so
    every rank raises the same InstabilityError (and none is left waiting in the next step's
    halo exchange)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(per_half)
    big = np.iinfo(np.int64).max
    dev = device if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([v if v >= 0 else big for v in per_half], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return [int(v) if int(v) != big else -1 for v in t.cpu()]


def raise_first_bad(per_half: list[int], grid: GridSpec, step_index) -> None:
    """Raise the reference's InstabilityError for the first half step with a bad node."""
    m1, m2, _ = grid.cells_per_axis
    for idx in per_half:
        if idx >= 0:
            raise InstabilityError(_node_of(idx, GridSpec((m1, m2, grid.cells_per_axis[2]))), step_index)


class SlabSolver:
    """Distributed full steps of a periodic field, one x3 slab per rank (one GPU per rank).

    Fields are stored with ghost planes (see module doc); `state` / `scratch`
    return views of the local planes.  Used by bench.py for the 2/4/8-GPU runs.
    """

    def __init__(self, global_cells, order_n: int, cfg: StepConfig, lengths=(1.0, 1.0, 1.0), group=None,
                 halo: str = "nccl"):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.grid = GridSpec(tuple(global_cells), tuple(lengths))
        self.order_n = order_n
        self.cfg = cfg
        m1, m2, m3 = self.grid.cells_per_axis
        self.z0, self.z1 = slab_bounds(m3, self.world, self.rank)
        self.local = self.z1 - self.z0
        if self.local < 2:
            raise ValueError("each rank needs at least two x3 planes")
        n = order_n + 1
        shape = (self.local + 2, m2, m1, n, n, n)
        self.bufs = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(2)]
        self.ops = OperatorSet.for_grid(self.grid, order_n)
        self.dt = select_dt(self.grid, cfg)
        self.flags = torch.full((2,), -1, dtype=torch.int64, device="cuda")
        self._guard = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        self.kernel_events = []
        q = cfg.stages(order_n)
        self._fac = _factor_arrays(self.ops, np.float64, self.dt / 2, q)
        self._q = q
        if halo not in ("nccl", "p2p", "auto"):
            raise ValueError(f"halo must be 'nccl', 'p2p' or 'auto', got {halo!r}")
        self.halo = halo
        self.halo_note = ""
        self._coeff = None  # two-pass coefficient chunk (allocated at the first half step)
        if cfg.mode == "two_pass":
            # the in-kernel p2p halo exists for the monolithic kernels; the two-kernel step reads
            # its ghost plane from the NCCL copy (recon_pass with periodic_z = 0)
            if halo == "p2p":
                raise ValueError("the p2p halo is implemented for the fused mode; use halo='nccl'")
            self.halo, self.halo_note = "nccl", ("two-kernel step: NCCL halo" if halo == "auto" else "")
        elif halo == "auto":
            # in-kernel p2p halo where it is available (N = 3, 5), verified against the NCCL copy
            # on the first initialised field (init); any failure falls back to NCCL
            if order_n in (3, 5):
                if not self._setup_p2p(tolerant=True):  # collective: all ranks agree
                    self.halo = "nccl"
            else:
                self.halo, self.halo_note = "nccl", "p2p halo kernels exist for N = 3, 5"
        elif halo == "p2p":
            self._setup_p2p()

    @property
    def launches_per_step(self) -> int:
        """Kernel launches per full step: one per half step with the in-kernel halo, two (interior
        + boundary plane) with the NCCL copy; the two-kernel step launches recon + evolve per
        coefficient chunk of each range."""
        if self.cfg.mode == "two_pass":
            chunk = self._coeff_planes()
            return 2 * 2 * (-(-(self.local - 1) // chunk) + 1)
        return 2 if self.halo == "p2p" else 4

    def _coeff_planes(self) -> int:
        from .pipeline import _coeff_chunk_planes
        m1, m2, _ = self.grid.cells_per_axis
        return _coeff_chunk_planes(GridSpec((m1, m2, self.local)), self.order_n, 8, self.cfg.coeff_budget_bytes)

    @property
    def state(self) -> torch.Tensor:
        return self.bufs[0][1:-1]

    @property
    def scratch(self) -> torch.Tensor:
        return self.bufs[1][1:-1]

    def init(self, ic) -> None:
        """Device initial data of this rank's planes (global x3 coordinates)."""
        from .problems import init_tables, launch_init
        t1, t2, t3 = init_tables(ic, self.grid, self.order_n)
        m1, m2, _ = self.grid.cells_per_axis
        tables = (t1, t2, np.ascontiguousarray(t3[:, self.z0:self.z1]))
        launch_init(self.state, (m1, m2, self.local), self.order_n, tables)
        if self.halo == "auto":
            self._verify_p2p()  # steps the field through both halo paths ...
            launch_init(self.state, (m1, m2, self.local), self.order_n, tables)  # ... so start over

    def _verify_p2p(self) -> None:
        """Both half steps (both neighbours' mappings) through both halo paths; all ranks must
        agree bit for bit, else the solver uses the NCCL copy from now on.  Memory-light (the
        fields fill HBM at 512^3 per GPU): the plane that reads the ghost is compared exactly,
        the whole field through a 64-bit checksum of its bits.  Leaves the fields stepped."""
        ok = True

        def attempt(fn):
            # a local failure must not skip the collectives inside the later steps (the halo
            # barrier / exchange): record it and carry on, the vote below decides for everyone
            nonlocal ok
            try:
                return fn()
            except Exception as exc:  # noqa: BLE001
                ok = False
                self.halo_note = self.halo_note or f"p2p verification raised: {exc}"
                return None

        flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        L = self.local
        for si, di, off, edge in ((0, 1, 0, L), (1, 0, -1, 1)):  # edge: buffer index of the ghost-reading plane
            attempt(lambda: self._half_p2p(si, di, off, flag, False))
            via_p2p = attempt(lambda: (self.bufs[di][1:-1].view(torch.int64).sum(), self.bufs[di][edge].clone()))
            attempt(lambda: self.half_step(self.bufs[si], self.bufs[di], off, flag))
            same = attempt(lambda: bool(via_p2p[0] == self.bufs[di][1:-1].view(torch.int64).sum())
                           and bool(torch.equal(via_p2p[1], self.bufs[di][edge])))
            ok = ok and bool(same)
            del via_p2p
        votes = torch.tensor([0.0 if ok else 1.0], device="cuda" if self.world == 1 or
                             dist.get_backend(self.group) == "nccl" else "cpu")
        if self.world > 1:
            dist.all_reduce(votes, group=self.group)
        if float(votes.item()) == 0.0:
            self.halo = "p2p"
        else:
            self.halo = "nccl"
            self.halo_note = self.halo_note or "p2p result differed from the NCCL halo"

    def _launch(self, src, dst, off, zb, ze, flag, events, guard=None):
        m1, m2, _ = self.grid.cells_per_axis
        h_mat, f1, f2, f3, cf = self._fac
        plane = src[0].numel() * src.element_size()
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True) if events is not None else None
        if e0 is not None:
            e0.record(stream)
        if self.cfg.mode == "two_pass":
            self._launch_two_pass(src, dst, off, zb, ze, flag, guard, plane, stream)
            if e0 is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                events.append((e0, e1))
            return
        rc = _native.lib().h3_fused_pass(
            ctypes.c_void_p(src.data_ptr() + plane), ctypes.c_void_p(dst.data_ptr() + plane),
            m1, m2, self.local, self.order_n, _ptr(h_mat), _ptr(f1), _ptr(f2), _ptr(f3), _ptr(cf),
            self._q, off, zb, ze, 0, _native.VARIANTS[self.cfg.variant], ctypes.c_void_p(stream.cuda_stream),
            ctypes.c_void_p(flag.data_ptr()), None if guard is None else ctypes.c_void_p(guard.data_ptr()))
        _native.check(rc, "h3_fused_pass (slab)")
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            events.append((e0, e1))

    def _launch_two_pass(self, src, dst, off, zb, ze, flag, guard, plane, stream):
        """The two-kernel half step of cells [zb, ze) of the slab (reference pipeline.py:254-273):
        reconstruction into a coefficient chunk -- reading the ghost plane at the slab edge
        (periodic_z = 0) -- then evolution, chunk by chunk."""
        m1, m2, _ = self.grid.cells_per_axis
        s = 2 * self.order_n + 2
        if self._coeff is None:
            self._coeff = torch.empty((self._coeff_planes(), m2, m1, s, s, s), dtype=torch.float64, device="cuda")
        h_mat, f1, f2, f3, cf = self._fac
        lib, var = _native.lib(), _native.VARIANTS[self.cfg.variant]
        sp, dp = ctypes.c_void_p(src.data_ptr() + plane), ctypes.c_void_p(dst.data_ptr() + plane)
        cp = ctypes.c_void_p(self._coeff.data_ptr())
        sh = ctypes.c_void_p(stream.cuda_stream)
        gp = None if guard is None else ctypes.c_void_p(guard.data_ptr())
        chunk = self._coeff.shape[0]
        for z0 in range(zb, ze, chunk):
            z1 = min(ze, z0 + chunk)
            _native.check(lib.h3_recon_pass(sp, cp, m1, m2, self.local, self.order_n, _ptr(h_mat), off, z0, z1, 0,
                                            var, sh, gp), "h3_recon_pass (slab)")
            _native.check(lib.h3_evolve_pass(cp, dp, m1, m2, self.local, self.order_n, _ptr(f1), _ptr(f2), _ptr(f3),
                                             _ptr(cf), self._q, z0, z1, var, sh, ctypes.c_void_p(flag.data_ptr()),
                                             gp), "h3_evolve_pass (slab)")

    # ---- p2p halo: the kernel reads the neighbour's boundary plane in place (CUDA IPC / NVLink) ----
    def _all_ranks_ok(self, ok: bool) -> bool:
        """Collective AND of a per-rank verdict (every rank must call it)."""
        if self.world == 1:
            return ok
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64,
                            device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return bool(flag.item())

    def _setup_p2p(self, tolerant: bool = False) -> bool:
        """Map the neighbours' field buffers (CUDA IPC handles exchanged through the process
        group); with one rank the 'neighbours' are the rank itself (periodic wrap).

        Collective and failure-consistent: every rank takes part in the handle exchange and in
        the final verdict even if its own export or mapping failed, so either all ranks use the
        p2p halo or none does (no rank is left waiting in a collective).  tolerant: report a
        failure by returning False (the caller falls back to NCCL) instead of raising."""
        lib = _native.lib()
        mine, err = None, None
        try:
            if self.order_n not in (3, 5):
                raise NotImplementedError("the in-kernel p2p halo is implemented for N = 3 and 5")
            mine = []
            for b in self.bufs:
                h = (ctypes.c_ubyte * 64)()
                off = ctypes.c_int64()
                _native.check(lib.h3_ipc_export(ctypes.c_void_p(b.data_ptr()), h, ctypes.byref(off)),
                              "h3_ipc_export")
                mine.append((bytes(h), int(off.value), self.local))
        except Exception as exc:  # noqa: BLE001 -- reported collectively below
            err = exc
        everyone = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(everyone, mine, group=self.group)
        else:
            everyone = [mine]
        self._opened = []
        bases = {}  # IPC handle -> mapped allocation base
        self._peer = {}  # rank -> ([buf0 ptr, buf1 ptr], local planes); ptr = the ghosted buffer base
        if err is None:
            try:
                for r in {(self.rank - 1) % self.world, (self.rank + 1) % self.world}:
                    if r == self.rank:
                        self._peer[r] = ([b.data_ptr() for b in self.bufs], self.local)
                        continue
                    if everyone[r] is None:
                        raise RuntimeError(f"rank {r} could not export its field buffers")
                    ptrs = []
                    for handle, offset, _ in everyone[r]:
                        if handle not in bases:  # both fields may live in one allocation: map it once
                            base = ctypes.c_void_p()
                            hb = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
                            _native.check(lib.h3_ipc_open(hb, ctypes.byref(base)), "h3_ipc_open")
                            self._opened.append(base.value)
                            bases[handle] = base.value
                        ptrs.append(bases[handle] + offset)
                    self._peer[r] = (ptrs, everyone[r][0][2])
            except Exception as exc:  # noqa: BLE001
                err = exc
        if not self._all_ranks_ok(err is None):
            self.close()
            self._peer = {}
            reason = f"p2p setup failed: {err}" if err is not None else "p2p setup failed on another rank"
            if tolerant:
                self.halo_note = reason
                return False
            raise RuntimeError(reason) from err
        self._sync = torch.zeros(1, device="cuda")
        return True

    def _barrier(self):
        """Stream-ordered rendezvous: every rank's previous half step is complete (its planes are
        final and nobody still reads the buffer about to be overwritten)."""
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._sync, group=self.group)
        else:  # gloo (tests: several ranks sharing one GPU)
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def _any_bad(self, flag: torch.Tensor) -> torch.Tensor:
        """Device guard for the second half step: != -1 when the first half step failed on ANY
        rank (all-reduce MAX of the signed flags; -1 = no bad node), so every rank skips it and
        leaves its state untouched, as the reference does after raising (pipeline.py:274).
        Stream-ordered under NCCL; it also orders the ranks' first half steps before the second
        (the p2p halo's rendezvous)."""
        if self.world == 1:
            return flag
        if dist.get_backend(self.group) == "nccl":
            self._guard.copy_(flag)
            dist.all_reduce(self._guard, op=dist.ReduceOp.MAX, group=self.group)
            return self._guard
        torch.cuda.synchronize()  # gloo (tests: several ranks sharing one GPU)
        host = flag.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.MAX, group=self.group)
        self._guard.copy_(host)
        return self._guard

    def _half_p2p(self, si, di, off, flag, timed, guard=None, collective_guard=False):
        """One p2p-halo half step.  collective_guard: `guard` is this rank's flag of the previous
        half step; the rendezvous becomes its all-reduce (_any_bad), one collective either way."""
        m1, m2, _ = self.grid.cells_per_axis
        h_mat, f1, f2, f3, cf = self._fac
        src, dst = self.bufs[si], self.bufs[di]
        plane = src[0].numel() * src.element_size()
        if collective_guard:
            guard = self._any_bad(guard)
        else:
            self._barrier()
        glo = ghi = None
        if off == 0:  # cell L-1 reads node plane L = rank+1's first local plane
            ptrs, _ = self._peer[(self.rank + 1) % self.world]
            ghi = ctypes.c_void_p(ptrs[si] + plane)
        else:         # cell 0 reads node plane -1 = rank-1's last local plane
            ptrs, lprev = self._peer[(self.rank - 1) % self.world]
            glo = ctypes.c_void_p(ptrs[si] + lprev * plane)
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True) if timed else None
        if e0 is not None:
            e0.record(stream)
        rc = _native.lib().h3_fused_pass_halo(
            ctypes.c_void_p(src.data_ptr() + plane), ctypes.c_void_p(dst.data_ptr() + plane), m1, m2, self.local,
            self.order_n, _ptr(h_mat), _ptr(f1), _ptr(f2), _ptr(f3), _ptr(cf), self._q, off, 0, self.local,
            glo, ghi, _native.VARIANTS[self.cfg.variant], ctypes.c_void_p(stream.cuda_stream),
            ctypes.c_void_p(flag.data_ptr()), None if guard is None else ctypes.c_void_p(guard.data_ptr()))
        _native.check(rc, "h3_fused_pass_halo")
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            self.kernel_events.append((e0, e1))

    def close(self) -> None:
        """Unmap the peer buffers (p2p halo)."""
        for base in getattr(self, "_opened", []):
            _native.lib().h3_ipc_close(ctypes.c_void_p(base))
        self._opened = []

    def half_step(self, src, dst, off, flag, timed=False, guard=None):
        works = exchange_halo(src, off, self.group, async_op=True)
        ev = self.kernel_events if timed else None
        L = self.local
        # interior cell planes first (they do not read the ghost plane) ...
        if off == 0:
            self._launch(src, dst, off, 0, L - 1, flag, ev, guard)
        else:
            self._launch(src, dst, off, 1, L, flag, ev, guard)
        for w in works:
            w.wait()  # current stream waits for the NCCL stream
        # ... then the boundary cell plane that does
        if off == 0:
            self._launch(src, dst, off, L - 1, L, flag, None, guard)
        else:
            self._launch(src, dst, off, 0, 1, flag, None, guard)

    def step(self, timed=False) -> None:
        """One full step.  Guard chain (as `run_steps`): the first half step is skipped when the
        previous step failed, the second when the first failed on any rank; flags are sticky, so
        after an instability the solver stops changing the fields until `clear_flags()`."""
        if self.halo == "auto":
            raise RuntimeError("call init() first (it selects the halo path)")
        f0, f1 = self.flags[0:1], self.flags[1:2]
        if self.halo == "p2p":
            self._half_p2p(0, 1, 0, f0, timed, guard=f1)
            self._half_p2p(1, 0, -1, f1, timed, guard=f0, collective_guard=True)
            return
        self.half_step(self.bufs[0], self.bufs[1], 0, f0, timed, guard=f1)
        self.half_step(self.bufs[1], self.bufs[0], -1, f1, timed, guard=self._any_bad(f0))

    def clear_flags(self) -> None:
        """Forget a reported instability (e.g. to retry from the untouched state with another dt)."""
        self.flags.fill_(-1)

    def check(self, step_index=None) -> None:
        """Raise InstabilityError on EVERY rank when any rank has produced a non-finite value
        (flags are sticky: call after each step; the first bad node over the whole grid, in
        half-step order)."""
        m1, m2, _ = self.grid.cells_per_axis
        plane = m1 * m2
        local = [int(b) + self.z0 * plane if int(b) != -1 else -1 for b in self.flags.cpu().numpy()]
        raise_first_bad(agree_first_bad(local, self.group, self.flags.device), self.grid, step_index)
