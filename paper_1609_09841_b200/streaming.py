"""Full steps of a HOST-resident field, streamed through the GPU in x3 chunks.

The reference steps a field that lives in host memory (numpy, pipeline.py:277-293).  The
drop-in equivalent with host buffers has to move the whole primary field to the GPU and back
every step; done naively (upload, step, download) that is two serial PCIe transfers per step.
`HostStepper` pipelines them instead: the primary field is cut into x3 chunks and, per step,

    upload chunk k                                            -> stream h2d
    dual chunk k      = half step off=0 of those planes       -> stream compute
    primary chunk k   = half step off=-1 of dual chunks k-1,k -> stream compute
    download primary chunk k                                  -> stream d2h

so uploads, kernels and downloads of different chunks overlap and a step costs about one
PCIe transfer time (both directions run concurrently).  The device holds only a few chunks,
so grids larger than HBM (e.g. 1024^3 at m = 3, 550 GB per field) can be stepped on one GPU.

Wrap-around (periodic x3): dual chunk K-1 needs primary plane 0, and primary chunk 0 needs dual
plane M3-1, so primary chunk 0 is finished last; its dual chunk is kept in a dedicated buffer
and a device copy of the original plane 0 serves as the ghost of chunk K-1.  The other ghost
planes are copied device to device from the next chunk's upload, so every primary plane crosses
PCIe exactly once in each direction.

Slabs (multi-GPU, one rank per GPU): with a torch.distributed process group of more than one
rank, each rank streams its own x3 slab of the global grid (`distributed.slab_bounds`) and the
two wrap-around planes become the slab halo: the rank's original first plane goes to rank-1
and rank+1's arrives as the ghost of the last dual chunk (one exchange at the start of the
step), and the last dual plane goes to rank+1 while rank-1's arrives as the ghost of primary
chunk 0 (one exchange before it is finished) -- NCCL send/recv on the compute stream.

Each chunk is a slab with ghost planes, stepped by the same C-ABI half step as the
single-field path (h3_fused_pass with periodic_z = 0), so results are bit-identical to
`full_step` on a device-resident field.  Instabilities raise the reference's
InstabilityError (same node and step); as the field is updated in place while streaming,
the host state is undefined after such an error.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .field import GridSpec
from .pipeline import InstabilityError, OperatorSet, StepConfig, _factor_arrays, _node_of, _ptr, select_dt

__all__ = ["chunk_plan", "HostStepper"]


def chunk_plan(m3: int, chunk: int, ramp: bool = False) -> list[tuple[int, int]]:
    """x3 chunks [z0, z1) covering 0..m3, each at least 2 planes (the ghost logic needs it).

    ramp: start and end with small chunks (chunk/8, /4, /2, then full ones, mirrored at the
    end), so the pipeline's fill (first upload, nothing to download yet) and drain (last
    downloads, nothing left to upload) are short."""
    if m3 < 2:
        raise ValueError("streaming needs at least two x3 planes")
    chunk = max(2, min(int(chunk), m3))
    sizes = []
    if ramp:
        head = [max(2, chunk >> s) for s in (3, 2, 1)]
        if 2 * sum(head) < m3:
            sizes = head
            tail = head[::-1]
            left = m3 - 2 * sum(head)
            sizes += [chunk] * (left // chunk) + ([left % chunk] if left % chunk else []) + tail
    if not sizes:
        sizes = [chunk] * (m3 // chunk) + ([m3 % chunk] if m3 % chunk else [])
    bounds, z = [], 0
    for size in sizes:
        bounds.append((z, z + size))
        z += size
    # fold chunks of fewer than 2 planes into their predecessor
    merged = []
    for z0, z1 in bounds:
        if merged and z1 - z0 < 2:
            merged[-1] = (merged[-1][0], z1)
        else:
            merged.append((z0, z1))
    if len(merged) > 1 and merged[0][1] - merged[0][0] < 2:
        merged[:2] = [(0, merged[1][1])]
    return merged


class HostStepper:
    """Streamed full steps of a pinned host field (M3, M2, M1, n, n, n), updated in place."""

    def __init__(self, host_state: torch.Tensor, grid: GridSpec, order_n: int, cfg: StepConfig | None = None,
                 chunk_planes: int | None = None, device=None, group=None, ramp: bool = True):
        """`grid` is the global grid.  Without a multi-rank process group `host_state` is the
        whole field (M3, M2, M1, n, n, n); with one (`group`, default: the default group when
        torch.distributed is initialised) it is this rank's slab (z1 - z0, M2, M1, n, n, n),
        [z0, z1) = distributed.slab_bounds(M3, world, rank)."""
        cfg = cfg or StepConfig()
        if cfg.mode != "fused" or cfg.precision != "double":
            raise ValueError("HostStepper streams the fused FP64 half step")
        m1, m2, m3 = grid.cells_per_axis
        n = order_n + 1
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 1:
            from .distributed import slab_bounds
            self.z0, z1 = slab_bounds(m3, self.world, self.rank)
            planes = z1 - self.z0
        else:
            self.z0, planes = 0, m3
        if host_state.device.type != "cpu" or tuple(host_state.shape) != (planes, m2, m1, n, n, n) \
                or host_state.dtype != torch.float64 or not host_state.is_contiguous():
            raise ValueError(f"host_state must be a contiguous CPU float64 tensor of shape "
                             f"{(planes, m2, m1, n, n, n)} (this rank's x3 planes, M2, M1, n, n, n)")
        self.host = host_state
        self.pinned = host_state.is_pinned()
        self.grid = grid.with_parity("primary")
        self.order_n = order_n
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ops = OperatorSet.for_grid(self.grid, order_n)
        plane = m1 * m2 * n ** 3
        if chunk_planes is None:  # ~2 GB chunks: measured best at 512^3 (tools/time_stream.py)
            chunk_planes = max(2, (2 << 30) // (plane * 8))
        self.chunks = chunk_plan(planes, chunk_planes, ramp=ramp)
        cmax = max(z1 - z0 for z0, z1 in self.chunks)
        kw = dict(dtype=torch.float64, device=self.device)
        shape = lambda planes: (planes, m2, m1, n, n, n)  # noqa: E731
        self.pin = [torch.empty(shape(cmax + 1), **kw) for _ in range(2)]    # chunk + next plane
        self.dbuf = [torch.empty(shape(cmax + 1), **kw) for _ in range(2)]   # ghost + dual chunk
        self.dual0 = torch.empty(shape(self.chunks[0][1] + 1), **kw)         # dual chunk 0 (kept)
        self.pout = [torch.empty(shape(cmax), **kw) for _ in range(2)]
        self.plane0 = torch.empty(shape(1)[1:], **kw)
        self.ghost_hi = torch.empty(shape(1)[1:], **kw) if self.world > 1 else self.plane0
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.h2d_bytes = planes * plane * 8
        self.d2h_bytes = planes * plane * 8
        self._plane = plane

    # -- one half step on a slab with ghost planes (h3_fused_pass, periodic_z = 0) --------------
    def _half(self, src_planes0: torch.Tensor, dst: torch.Tensor, planes: int, off: int, fac, flag):
        m1, m2, _ = self.grid.cells_per_axis
        h_mat, f1, f2, f3, cf = fac
        rc = _native.lib().h3_fused_pass(
            ctypes.c_void_p(src_planes0.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
            m1, m2, planes, self.order_n, _ptr(h_mat), _ptr(f1), _ptr(f2), _ptr(f3), _ptr(cf),
            self.cfg.stages(self.order_n), off, 0, planes, 0, _native.VARIANTS[self.cfg.variant],
            ctypes.c_void_p(self.s_cmp.cuda_stream), ctypes.c_void_p(flag.data_ptr()), None)
        _native.check(rc, "h3_fused_pass (streamed chunk)")

    def _swap(self, send: torch.Tensor, send_to: int, recv: torch.Tensor, recv_from: int) -> None:
        """Send one plane to a neighbour rank and receive one, ordered on the compute stream."""
        g = self.group
        to_g = dist.get_global_rank(g, send_to) if g is not None else send_to
        from_g = dist.get_global_rank(g, recv_from) if g is not None else recv_from
        if dist.get_backend(g) == "gloo":  # host staging (tests of the multi-rank path on one GPU)
            host_send, host_recv = send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, host_send, to_g, g),
                                             dist.P2POp(dist.irecv, host_recv, from_g, g)]):
                w.wait()
            recv.copy_(host_recv)
            return
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, send, to_g, g),
                                         dist.P2POp(dist.irecv, recv, from_g, g)]):
            w.wait()  # NCCL: makes the current (compute) stream wait, not the host

    def step(self, dt: float | None = None, step_index: int | None = None) -> None:
        """One full step (primary -> dual -> primary) of the host field, in place."""
        if dt is None:
            dt = select_dt(self.grid, self.cfg)
        fac = _factor_arrays(self.ops, np.float64, dt / 2, self.cfg.stages(self.order_n))
        m3 = self.grid.cells_per_axis[2]
        K = len(self.chunks)
        flags = torch.full((2, K), -1, dtype=torch.int64, device=self.device)
        nb = self.pinned
        ev = lambda: torch.cuda.Event()  # noqa: E731
        pin_free = [None, None]    # compute finished reading pin[i]
        pout_free = [None, None]   # download finished reading pout[i]
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)

        def upload(k):
            z0, z1 = self.chunks[k]
            L = z1 - z0
            buf = self.pin[k % 2]
            with torch.cuda.stream(self.s_h2d):
                if pin_free[k % 2] is not None:
                    self.s_h2d.wait_event(pin_free[k % 2])
                buf[:L].copy_(self.host[z0:z1], non_blocking=nb)
                if k == 0:  # original plane 0: the ghost of the last dual chunk (wrap)
                    self.plane0.copy_(buf[0])
                e = ev()
                e.record(self.s_h2d)
            return e

        def finish(k, dsrc: torch.Tensor):
            """primary chunk k from dual planes z0-1 .. z1-1 held in dsrc[0 .. L]; then download."""
            z0, z1 = self.chunks[k]
            L = z1 - z0
            out = self.pout[k % 2]
            with torch.cuda.stream(self.s_cmp):
                if pout_free[k % 2] is not None:
                    self.s_cmp.wait_event(pout_free[k % 2])
                self._half(dsrc[1:], out, L, -1, fac, flags[1, k])
                done = ev()
                done.record(self.s_cmp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done)
                self.host[z0:z1].copy_(out[:L], non_blocking=nb)
                e = ev()
                e.record(self.s_d2h)
                pout_free[k % 2] = e

        up = upload(0)
        nxt_rank, prv_rank = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        if self.world > 1:  # my original first plane -> rank-1, rank+1's -> ghost of the last dual chunk
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(up)
                self._swap(self.plane0, prv_rank, self.ghost_hi, nxt_rank)
        for k in range(K):
            nxt = upload(k + 1) if k + 1 < K else None
            z0, z1 = self.chunks[k]
            L = z1 - z0
            dst = self.dual0 if k == 0 else self.dbuf[k % 2]
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(up)
                # high ghost plane = first plane of chunk k+1 (already on the device), or the
                # original plane 0 for the last chunk: each primary plane crosses PCIe once
                if nxt is not None:
                    self.s_cmp.wait_event(nxt)
                    self.pin[k % 2][L].copy_(self.pin[(k + 1) % 2][0])
                else:
                    self.pin[k % 2][L].copy_(self.ghost_hi)
                self._half(self.pin[k % 2], dst[1:], L, 0, fac, flags[0, k])
                e = ev()
                e.record(self.s_cmp)
                pin_free[k % 2] = e
                if k >= 1:  # ghost plane: last dual plane of chunk k-1
                    prev = self.dual0 if k == 1 else self.dbuf[(k - 1) % 2]
                    lp = self.chunks[k - 1][1] - self.chunks[k - 1][0]
                    dst[0].copy_(prev[lp])
            if k >= 1:
                finish(k, dst)
            up = nxt
        # primary chunk 0 last: its ghost is the last dual plane of chunk K-1 (of rank-1 for slabs)
        with torch.cuda.stream(self.s_cmp):
            last = self.dual0 if K == 1 else self.dbuf[(K - 1) % 2]
            lp = self.chunks[K - 1][1] - self.chunks[K - 1][0]
            if self.world > 1:
                self._swap(last[lp], nxt_rank, self.dual0[0], prv_rank)
            else:
                self.dual0[0].copy_(last[lp])
        finish(0, self.dual0)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            cur.wait_stream(s)
        host_flags = flags.cpu().numpy()  # the step's result read back (synchronises)
        self._raise(host_flags, step_index)

    def _raise(self, host_flags, step_index):
        m1, m2, _ = self.grid.cells_per_axis
        per_half = []
        for half in (0, 1):  # dual, then primary: the reference raises after the first bad half step
            best = -1
            for k, (z0, _z1) in enumerate(self.chunks):
                bad = int(host_flags[half, k])
                if bad != -1:
                    idx = bad + (z0 + self.z0) * m1 * m2  # chunk-local C-order index -> global
                    best = idx if best == -1 else min(best, idx)
            per_half.append(best)
        if self.world > 1:
            from .distributed import agree_first_bad
            per_half = agree_first_bad(per_half, self.group, self.device)
        for idx in per_half:
            if idx != -1:
                raise InstabilityError(node=_node_of(idx, self.grid), step=step_index)
