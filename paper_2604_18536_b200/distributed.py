"""Multi-GPU z-slab decomposition of the RK4 time-step path.

The periodic box is split along axis 0 (the slowest storage axis -- the
survey's "z" in its [z][y][x] naming) into P slabs of m = n0/P planes, one
process per GPU (``torch.distributed``, NCCL over NVLink).  Per projection:

    halo(u)            exchange the +-1 ghost planes of u with the neighbours
    r2c                divergence -> R2C (axis 2)
    per column chunk:  FFT axis 1 -> all_to_all (m, n1, w) -> (n0, n1/P, w)
                       -> FFT axis 0 -> 1/(Lambda N) -> inverse FFT axis 0
                       -> all_to_all back -> inverse FFT axis 1 (pipelined)
    c2r                C2R (local pressure)
    p halo             next slab's first pressure plane
    correct            u -= G p, ghost fill of axes 1, 2
    halo(u)            for the next stencil

The RHS stencils reach +-1 plane, so the fused RK-stage kernel only needs the
ghost planes exchanged after every projection.  Kinetic energy and CFL use
an all-reduce.  The reference is single-process; this
is the paper's outlook built B200-first.

The local compute is a ``backend`` object: ``CudaSlabBackend`` calls the C
ABI (``sfb_slab_*``, ``sfb_rk_stage``); the CPU gloo tests plug in a numpy
backend so the orchestration (slab bookkeeping, halo directions, all-to-all
packing) is exercised with world_size 2 on CPU.
"""

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .fields import VelocityField
from .grid import AxisCoords, Grid


class SlabLayout:
    """Which planes of axis 0 this rank owns (host bookkeeping only)."""

    def __init__(self, n0, rank, size):
        if n0 % size:
            raise ValueError(f"n0={n0} must be divisible by the number of ranks {size}")
        self.n0, self.rank, self.size = n0, rank, size
        self.m = n0 // size
        self.i0 = rank * self.m  # first owned interior plane is global index i0 + 1
        self.prev = (rank - 1) % size
        self.next = (rank + 1) % size

    def global_planes(self):
        return range(self.i0 + 1, self.i0 + self.m + 1)


class SlabGrid(Grid):
    """The local slab of a global grid: axis-0 tables sliced from the global
    extended tables (ghost widths are the neighbours' widths)."""

    def __init__(self, global_grid, layout):
        g = global_grid
        m, i0 = layout.m, layout.i0
        b0 = g.axes[0].boundaries[i0:i0 + m + 1]
        super().__init__((AxisCoords(b0),) + tuple(g.axes[1:]), g.periodic, dtype=g.dtype)
        self.global_grid = g
        self.layout = layout
        sl = slice(i0, i0 + m + 2)
        self.dx = [g.dx[0][sl].copy()] + list(g.dx[1:])
        self.du = [g.du[0][sl].copy()] + list(g.du[1:])
        self.xb = [g.xb[0][sl].copy()] + list(g.xb[1:])
        self.xc = [g.xc[0][sl].copy()] + list(g.xc[1:])

    def packed_tables(self):
        if self._packed is None:
            full = self.global_grid.packed_tables()
            g = self.global_grid
            E0 = g.shape[0] + 2
            i0, m = self.layout.i0, self.layout.m
            parts = [full[t * E0 + i0: t * E0 + i0 + m + 2] for t in range(N.SFB_NTAB)]
            parts.append(full[N.SFB_NTAB * E0:])
            self._packed = np.ascontiguousarray(np.concatenate(parts))
        return self._packed


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------
class _Done:
    def wait(self):
        return True


class Comm:
    """Halo exchange, all-to-all and all-reduce over a process group.
    ``stage_host=True`` stages CUDA tensors through host memory (gloo)."""

    def __init__(self, layout, group=None, stage_host=False):
        self.layout = layout
        self.group = group
        self.stage_host = stage_host

    def _send_recv(self, send, recv, dst, src):
        if self.layout.size == 1:
            recv.copy_(send)
            return
        s = send.cpu() if self.stage_host else send.contiguous()
        r = torch.empty_like(s) if self.stage_host else recv
        ops = [dist.P2POp(dist.isend, s, dst, self.group), dist.P2POp(dist.irecv, r, src, self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if self.stage_host:
            recv.copy_(r)

    def halo(self, tensors):
        """Ghost planes along axis 0: plane 0 <- prev's last plane,
        plane m+1 <- next's first plane (all tensors' planes in one batch of
        P2P operations over NCCL)."""
        lay = self.layout
        m = lay.m
        if lay.size == 1 or self.stage_host:
            for t in tensors:
                self._send_recv(t[m], t[0], lay.next, lay.prev)
                self._send_recv(t[1], t[m + 1], lay.prev, lay.next)
            return
        ops = []
        for t in tensors:
            ops.append(dist.P2POp(dist.isend, t[m], lay.next, self.group))
            ops.append(dist.P2POp(dist.irecv, t[0], lay.prev, self.group))
            ops.append(dist.P2POp(dist.isend, t[1], lay.prev, self.group))
            ops.append(dist.P2POp(dist.irecv, t[m + 1], lay.next, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def plane_from_next(self, send_plane, recv_plane):
        self._send_recv(send_plane, recv_plane, self.layout.prev, self.layout.next)

    def plane_from_prev(self, send_plane, recv_plane):
        self._send_recv(send_plane, recv_plane, self.layout.next, self.layout.prev)

    def all_to_all(self, out, inp):
        self.all_to_all_async(out, inp).wait()

    def all_to_all_async(self, out, inp):
        """Equal-split all-to-all over dim 0; returns a handle whose wait()
        orders later work on the current stream after the exchange (NCCL:
        the exchange runs on NCCL's stream, overlapping the caller's next
        kernels)."""
        if self.layout.size == 1:
            out.copy_(inp)
            return _Done()
        if self.stage_host:
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
            return _Done()
        return dist.all_to_all_single(out, inp, group=self.group, async_op=True)

    def allreduce(self, value, op="sum"):
        if self.layout.size == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64)
        if not self.stage_host and torch.cuda.is_available() and dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MIN, group=self.group)
        return float(t.item())


class _Event:
    """Handle of an exchange enqueued on the communicator's stream: wait()
    orders the caller's current stream after it."""

    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)
        return True


class NcclComm:
    """The same operations as ``Comm`` through the library's own NCCL
    communicator (``sfb_comm_*`` in the C ABI): the halo planes of all
    fields in one NCCL group on the compute stream, the transposes'
    all-to-alls on a dedicated stream (ordered by CUDA events, so they
    overlap the next chunk's kernels), device-side fp64 all-reduces.  The
    128-byte NCCL id is broadcast over ``group`` (any torch.distributed
    backend); with one rank everything is a device copy."""

    def __init__(self, layout, group=None):
        import os

        # NCCL prints its version banner to stdout at the first init unless
        # told otherwise; keep stdout for the caller (bench.py's JSON line)
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        self.layout = layout
        id_buf = (ctypes.c_ubyte * 128)()
        if layout.rank == 0:
            N.call("sfb_comm_unique_id", ctypes.cast(id_buf, ctypes.c_void_p))
        if layout.size > 1:
            t = torch.tensor(list(id_buf), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            for i, b in enumerate(t.cpu().tolist()):
                id_buf[i] = b
        h = ctypes.c_void_p()
        N.call("sfb_comm_create", ctypes.cast(id_buf, ctypes.c_void_p), layout.size, layout.rank, ctypes.byref(h))
        self.handle = h
        self.stream = torch.cuda.Stream()
        self._red = torch.zeros(1, dtype=torch.float64, device="cuda")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib.sfb_comm_destroy(h)
            except Exception:  # pragma: no cover
                pass

    @staticmethod
    def _sp(stream=None):
        return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)

    def halo(self, tensors):
        m = self.layout.m
        t0 = tensors[0]
        ptrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in tensors] + [None] * (3 - len(tensors)))
        N.call("sfb_comm_halo", self.handle, ptrs, len(tensors), t0[0].numel() * t0.element_size(), m, self._sp())

    def _sendrecv(self, send, dst, recv, src):
        N.call("sfb_comm_sendrecv", self.handle, send.data_ptr(), dst, recv.data_ptr(), src,
               send.numel() * send.element_size(), self._sp())

    def plane_from_next(self, send_plane, recv_plane):
        lay = self.layout
        self._sendrecv(send_plane, lay.prev, recv_plane, lay.next)

    def plane_from_prev(self, send_plane, recv_plane):
        lay = self.layout
        self._sendrecv(send_plane, lay.next, recv_plane, lay.prev)

    def all_to_all(self, out, inp):
        self.all_to_all_async(out, inp).wait()

    def all_to_all_async(self, out, inp):
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        N.call("sfb_comm_alltoall", self.handle, inp.data_ptr(), out.data_ptr(),
               inp.numel() * inp.element_size() // self.layout.size, self._sp(self.stream))
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return _Event(ev)

    def allreduce_device(self, t, op="sum"):
        """In-place all-reduce of an fp64 CUDA tensor, no host round trip."""
        N.call("sfb_comm_allreduce_f64", self.handle, t.data_ptr(), t.numel(), {"sum": 0, "min": 1, "max": 2}[op],
               self._sp())
        return t

    def allreduce(self, value, op="sum"):
        if self.layout.size == 1:
            return value
        self._red.fill_(value)
        return float(self.allreduce_device(self._red, op).item())


def make_comm(layout, group=None):
    """The slab communicator of a CUDA run: the library's NCCL communicator
    (``SFB_COMM=torch`` keeps torch.distributed's)."""
    import os

    if os.environ.get("SFB_COMM", "nccl") == "torch":
        return Comm(layout, group=group)
    return NcclComm(layout, group=group)


# ---------------------------------------------------------------------------
# CUDA backend (C ABI)
# ---------------------------------------------------------------------------
class _DevBuf:
    """__cuda_array_interface__ view of a buffer owned by the native solver."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class CudaSlabBackend:
    def __init__(self, slab_grid, nu, force):
        from .bcs import BoundarySpec, Periodic

        from .plan import Plan

        g = slab_grid
        lay = g.layout
        n0, n1, n2 = g.global_grid.shape
        if n1 % lay.size:
            raise ValueError("n1 must be divisible by the number of ranks")
        self.grid = g
        self.nu = float(nu)
        self.force = [float(g.dtype.type(f)) for f in (force or (0.0, 0.0, 0.0))]
        bcs = BoundarySpec.all_periodic(3)
        self.plan = Plan(g, bcs, halo_axis0=True)
        h = ctypes.c_void_p()
        N.call("sfb_slab_solver_create", self.plan.handle, n0, lay.rank, lay.size, ctypes.byref(h))
        self.handle = h
        spec, trans, xchg, ps, pl, ph = (ctypes.c_void_p() for _ in range(6))
        N.call("sfb_slab_buffers", h, ctypes.byref(spec), ctypes.byref(trans), ctypes.byref(xchg), ctypes.byref(ps),
               ctypes.byref(pl), ctypes.byref(ph))
        ts = "<f8" if g.dtype == np.float64 else "<f4"
        m, nh = lay.m, n2 // 2 + 1
        P = lay.size
        self.spec = torch.as_tensor(_DevBuf(spec.value, (m, n1, nh, 2), ts), device="cuda")
        self.trans = torch.as_tensor(_DevBuf(trans.value, (n0, n1 // P, nh, 2), ts), device="cuda")
        # all-to-all send / receive buffer in the chunked layout (P, m, n1/P, nh)
        self.xchg = (torch.as_tensor(_DevBuf(xchg.value, (P, m, n1 // P, nh, 2), ts), device="cuda")
                     if P > 1 else None)
        # slab pressure: [prev's last | m local | next's first two] planes
        self.p_slab = torch.as_tensor(_DevBuf(ps.value, (m + 3, n1, n2), ts), device="cuda")
        self.p_local = self.p_slab[1:m + 1]
        self.p_halo = self.p_slab[m + 1]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib.sfb_solver_destroy(h)
            except Exception:  # pragma: no cover
                pass

    def _sp(self):
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def stage(self, y, u0=None, s_in=None, s_out=None, y_next=None, cb=0.0, ca=0.0, p_slab=None, u0_out=None):
        a = N.StageArgs()
        a.p_int = None if p_slab is None else p_slab.data_ptr()
        if u0_out is not None:
            a.u0_out = N.ptr3(u0_out.u)
        a.y = N.ptr3(y.u)
        a.u0 = N.ptr3(u0.u if u0 is not None else [None] * 3)
        a.s_in = N.ptr3(s_in.u if s_in is not None else [None] * 3)
        a.s_out = N.ptr3(s_out.u if s_out is not None else [None] * 3)
        a.y_next = N.ptr3(y_next.u if y_next is not None else [None] * 3)
        a.k_out = N.ptr3([None] * 3)
        a.cb, a.ca, a.nu = float(cb), float(ca), self.nu
        for i, f in enumerate(self.force):
            a.force[i] = f
        from . import timestep as TS

        if TS.STAGE_EVENTS is None:
            N.call("sfb_rk_stage", self.plan.handle, ctypes.byref(a), self._sp())
            return
        nfield = 1 + (s_out is not None) + (y_next is not None) + (u0_out is not None)
        nfield += (u0 is not None and u0 is not y and (y_next is not None or (s_out is not None and s_in is None)))
        nfield += (s_in is not None and s_out is not None)
        nfield += (1.0 / 3.0) if p_slab is not None else 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("sfb_rk_stage", self.plan.handle, ctypes.byref(a), self._sp())
        e1.record()
        TS.STAGE_EVENTS.append((e0, e1, nfield * 3 * self.grid.dtype.itemsize))

    def max_chunks(self):
        return int(N.lib.sfb_slab_max_chunks(self.handle))

    def r2c(self, u):
        N.call("sfb_slab_r2c", self.handle, N.ptr3(u.u), self._sp())

    def axis1(self, k, nchunks, inverse=False):
        N.call("sfb_slab_axis1", self.handle, int(k), int(nchunks), 1 if inverse else 0, self._sp())

    def axis0(self, k=0, nchunks=1):
        N.call("sfb_slab_axis0", self.handle, int(k), int(nchunks), self._sp())

    def c2r(self):
        N.call("sfb_slab_c2r", self.handle, self._sp())

    def correct(self, u, p_ext=None):
        N.call("sfb_slab_correct", self.handle, N.ptr3(u.u), None if p_ext is None else p_ext.data.data_ptr(), self._sp())

    def kinetic_energy_local(self, u):
        out = ctypes.c_double()
        N.call("sfb_kinetic_energy", self.plan.handle, N.ptr3(u.u), ctypes.byref(out), self._sp())
        return out.value

    def new_field(self):
        return VelocityField(self.grid)

    def new_scalar(self):
        from .fields import ScalarField

        return ScalarField(self.grid)


# ---------------------------------------------------------------------------
# orchestration (backend-agnostic)
# ---------------------------------------------------------------------------
class SlabProjector:
    """One projection of the slab-decomposed field.

    The half-spectrum columns are split into K chunks.  The axis-1 transform
    of chunk k writes its all-to-all send block directly (``xchg`` block k,
    laid out (P, m, n1/P, w_k)), so the exchange needs no packing, and the
    chunks are pipelined: the exchange of chunk k runs on NCCL's stream
    while chunk k+1 is transformed, the axis-0 solve of chunk k while the
    exchanges of later chunks are in flight, and so on.  With one rank there
    is no exchange at all."""

    def __init__(self, backend, comm, chunks=None):
        import os

        self.b = backend
        self.comm = comm
        if chunks is None:
            chunks = int(os.environ.get("SFB_SLAB_CHUNKS", "4"))
        self.K = max(1, min(chunks, backend.max_chunks())) if comm.layout.size > 1 else 1

    def _blocks(self):
        """(xchg block, trans block) views of chunk k, flat per rank."""
        b, lay = self.b, self.comm.layout
        P, m = lay.size, lay.m
        n0, c, nh = b.trans.shape[0], b.trans.shape[1], b.trans.shape[2]
        xf = b.xchg.reshape(-1)
        tf = b.trans.reshape(-1)
        base = (nh + self.K - 1) // self.K
        out = []
        for k in range(self.K):
            c0 = k * base
            w = min(base, nh - c0)
            if w <= 0:
                out.append(None)
                continue
            off, n = 2 * P * m * c * c0, 2 * P * m * c * w
            out.append((xf[off:off + n].view(P, -1), tf[off:off + n].view(P, -1)))
        return out

    def _solve(self, u):
        b, comm = self.b, self.comm
        P = comm.layout.size
        comm.halo(u.u)
        b.r2c(u)
        if P == 1:
            b.axis1(0, 1)
            b.axis0(0, 1)
            b.axis1(0, 1, inverse=True)
        else:
            K = self.K
            blocks = self._blocks()
            fwd = [None] * K
            for k in range(K):
                if blocks[k] is None:
                    continue
                b.axis1(k, K)
                fwd[k] = comm.all_to_all_async(blocks[k][1], blocks[k][0])
            back = [None] * K
            for k in range(K):
                if blocks[k] is None:
                    continue
                fwd[k].wait()
                b.axis0(k, K)
                back[k] = comm.all_to_all_async(blocks[k][0], blocks[k][1])
            for k in range(K):
                if blocks[k] is None:
                    continue
                back[k].wait()
                b.axis1(k, K, inverse=True)
        b.c2r()

    def project(self, u, p_ext=None):
        """Full projection (poisson.py:321-341) of the slab field."""
        b, comm = self.b, self.comm
        self._solve(u)
        comm.plane_from_next(b.p_local[0], b.p_halo)
        b.correct(u, p_ext)
        comm.halo(u.u)
        if p_ext is not None:
            comm.halo([p_ext.data])

    def finish(self, u, p_ext=None):
        """Complete a projection stopped after project_solve (u -= G p, ghost
        fills, halo): the tail of ``project``."""
        b, comm = self.b, self.comm
        b.correct(u, p_ext)
        comm.halo(u.u)
        if p_ext is not None:
            comm.halo([p_ext.data])

    def project_solve(self, u):
        """Projection split at the gradient subtract (timestep._project_solve):
        u keeps its exchanged (unprojected) ghost planes, the slab pressure
        gets the neighbours' planes the next stage kernel's y - G p needs
        (prev's last, next's first two); returns it."""
        b, comm = self.b, self.comm
        m = comm.layout.m
        self._solve(u)
        ps = b.p_slab
        comm.plane_from_next(ps[1], ps[m + 1])
        comm.plane_from_next(ps[2], ps[m + 2])
        comm.plane_from_prev(ps[m], ps[0])
        return ps


class SlabState:
    def __init__(self, u, regs, p, t=0.0):
        self.u = u
        self.regs = regs
        self.pressure = p
        self.t = t
        self.step = 0
        # run_steps: the last projection of the previous step stopped after
        # its solve (u unprojected, this slab pressure pending)
        self.pending = None


class SlabSimulation:
    """RK4 on a slab-decomposed periodic box (the fused 4-register scheme of
    timestep.rk_step, with the slab projector between stages; intermediate
    projections hand their pressure to the next stage kernel)."""

    def __init__(self, backend, comm):
        self.b = backend
        self.comm = comm
        self.proj = SlabProjector(backend, comm)

    def new_state(self, u_local):
        regs = [self.b.new_field() for _ in range(3)]
        p = self.b.new_scalar()
        self.comm.halo(u_local.u)
        return SlabState(u_local, regs, p)

    def rk4_step(self, state, dt, defer=False):
        """One RK4 step.  ``defer`` (run_steps): the step's last projection
        stops after its solve and the next step's stage 0 applies u - G p
        while staging u, writing the projected u0 once (timestep.rk_step's
        deferred form on the slab)."""
        from .timestep import RK4

        tab = RK4
        p_in = state.pending
        state.pending = None
        if p_in is not None:
            # registers: u* (the unprojected state), u0 (its projection), s, y
            u_star = state.u
            u0, acc, y = state.regs
            yn = None
        else:
            u_star = None
            u0 = state.u
            acc, y, yn = state.regs
        started = False
        cur = u0 if p_in is None else u_star
        p_pending = p_in
        for j in range(tab.stages):
            bj = tab.b[j]
            nxt = j + 1 < tab.stages
            if j == 0 and p_in is not None:
                self.b.stage(u_star, u0=u_star, s_out=acc, y_next=y, cb=dt * bj, ca=dt * tab.a[1][0],
                             p_slab=p_in, u0_out=u0)
                started = True
                yn = u_star  # u* is free once its projection is in u0
                p_pending = self.proj.project_solve(y)
                cur = y
                continue
            self.b.stage(cur, u0=u0, s_in=acc if started else None, s_out=acc if bj != 0.0 else None,
                         y_next=yn if nxt else None, cb=dt * bj, ca=dt * (tab.a[j + 1][j] if nxt else 0.0),
                         p_slab=p_pending)
            started = started or bj != 0.0
            if nxt:
                # intermediate projection split at the gradient subtract: the
                # next stage kernel forms y - G p from the slab pressure
                p_pending = self.proj.project_solve(yn)
                y, yn = yn, y
                cur = y
        if defer:
            state.pending = self.proj.project_solve(acc)
        else:
            self.proj.project(acc, p_ext=state.pressure)
        state.regs = [u0, y, yn]
        state.u = acc
        state.t += dt
        state.step += 1
        return state

    def finish(self, state):
        """Complete a deferred last projection (the state rk4_step returns)."""
        if state.pending is not None:
            self.proj.finish(state.u, p_ext=state.pressure)
            state.pending = None
        return state

    def run_steps(self, state, nsteps, dt):
        """timestep.run_steps on the slab: each step's last projection is
        finished by the next step's first stage kernel; the returned state is
        fully projected."""
        for _ in range(nsteps):
            self.rk4_step(state, dt, defer=True)
        return self.finish(state)

    def kinetic_energy(self, u):
        return self.comm.allreduce(self.b.kinetic_energy_local(u), "sum")


def scatter_field(global_arrays, layout):
    """Local extended slabs (with ghost planes) of global extended arrays."""
    m, i0 = layout.m, layout.i0
    return [np.ascontiguousarray(a[i0:i0 + m + 2]) for a in global_arrays]
