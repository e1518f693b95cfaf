"""Stepping trajectories whose velocity lives in host memory.

The reference keeps every field in host (numpy) arrays: a caller that holds
its states on the host and wants them advanced calls ``rk_step`` on each
(timestep.py:175-214) and reads the result back.  On the GPU that round trip
moves the whole extended velocity over PCIe twice per step (14.3 GB each way
at 840^3 fp64), which costs twice as long as the step itself.

``HostEnsemble`` keeps that contract -- each member's velocity is uploaded
from its pinned host buffer before each step and read back into it after --
but schedules the copies so they hide behind compute:

* uploads run on one copy stream, read-backs on another (PCIe is full
  duplex), in plane chunks; chunk c of a member's next upload waits only for
  chunk c of its read-back;
* members are stepped in turn on the compute stream, so member m's
  read-back and re-upload overlap the steps of the other members;
* all members share one ``Workspace`` (the RK registers and solver buffers
  are scratch within a step), so each extra member costs one velocity field
  of HBM.

Every member gets exactly the device step ``rk_step`` / ``wray3_step``
would give it (same kernels, same order; ghosts refilled after each upload
so host-side edits of the interior are honoured).  The host buffers hold
the results once ``synchronize()`` returns.
"""

import torch

from .errors import ConfigurationError
from .fields import VelocityField, fill_ghosts_velocity
from .timestep import SimState, _finish_pending, _step


class HostEnsemble:
    """Advance independent trajectories held in pinned host memory.

    ``host`` is a list of members, each a list of ``grid.dim`` pinned CPU
    tensors with the extended shape ``grid.ext_shape`` and the grid's dtype
    (the reference's extended array layout).  ``chunks`` plane chunks per
    component are copied at a time.
    """

    def __init__(self, setup, host, t0=0.0, chunks=8, state=None):
        if not host:
            raise ValueError("HostEnsemble needs at least one member")
        g = setup.grid
        for m, comps in enumerate(host):
            if len(comps) != g.dim:
                raise ValueError(f"member {m}: expected {g.dim} components, got {len(comps)}")
            for c in comps:
                if c.device.type != "cpu" or tuple(c.shape) != tuple(g.ext_shape) or c.dtype != _torch_dtype(g):
                    raise ValueError(f"member {m}: host components must be CPU tensors of shape "
                                     f"{tuple(g.ext_shape)} and the grid's dtype")
                if not c.is_pinned():
                    raise ConfigurationError("HostEnsemble needs pinned host buffers (torch.empty(..., pin_memory=True))")
        self.setup = setup
        self.host = host
        # member 0 may reuse an existing state (its workspace and velocity)
        base = state if state is not None else setup.new_state(t0=t0)
        _finish_pending(base, setup)  # a deferred projection must not meet an upload
        ws = base.workspace
        self.states = [base] + [SimState(u=VelocityField(g, empty=True), t=base.t, workspace=ws)
                                for _ in range(len(host) - 1)]
        n0 = g.ext_shape[0]
        chunks = max(1, min(int(chunks), n0))
        bounds = [round(c * n0 / chunks) for c in range(chunks + 1)]
        self._slices = [(a, slice(bounds[c], bounds[c + 1])) for a in range(g.dim) for c in range(chunks)]
        self._d2h = torch.cuda.Stream()
        self._h2d = torch.cuda.Stream()
        self._back = [[torch.cuda.Event() for _ in self._slices] for _ in host]  # read-back of chunk landed
        self._up = [torch.cuda.Event() for _ in host]                            # member uploaded
        self._fresh = [True] * len(host)  # upload not yet issued for the next step
        self.steps = 0

    def _upload(self, m):
        # chunk c waits for chunk c of this member's previous read-back (same
        # host and device buffers); before the first read-back the events are
        # unrecorded and the waits are no-ops
        st = self.states[m]
        with torch.cuda.stream(self._h2d):
            for (a, sl), ev in zip(self._slices, self._back[m]):
                self._h2d.wait_event(ev)
                st.u.u[a][sl].copy_(self.host[m][a][sl], non_blocking=True)
            self._up[m].record(self._h2d)
        self._fresh[m] = False

    def step(self, dt, last=False):
        """One step of every member: (upload ->) step -> read back.  With
        ``last`` the members' next uploads are not issued."""
        main = torch.cuda.current_stream()
        if any(self._fresh):
            # a fresh upload overwrites a member's device velocity: after
            # everything already queued on the compute stream
            self._h2d.wait_stream(main)
        for m in range(len(self.states)):
            if self._fresh[m]:
                self._upload(m)
        for m, st in enumerate(self.states):
            main.wait_event(self._up[m])
            fill_ghosts_velocity(st.u, self.setup.bcs, st.t)
            _step(st, dt, self.setup)
            self._d2h.wait_stream(main)
            with torch.cuda.stream(self._d2h):
                for (a, sl), ev in zip(self._slices, self._back[m]):
                    self.host[m][a][sl].copy_(st.u.u[a][sl], non_blocking=True)
                    ev.record(self._d2h)
            if last:
                self._fresh[m] = True
            else:
                self._upload(m)
        # Buffer rotation is safe without a join: a member's result buffer
        # leaves the workspace, its re-upload waits for its read-back, and its
        # next step waits for the re-upload -- so a read-back always finishes
        # before the buffer rotates back into the shared registers.
        self.steps += 1

    def run(self, n_steps, dt):
        """``n_steps`` steps of every member; host buffers hold the results
        after ``synchronize()``."""
        for i in range(n_steps):
            self.step(dt, last=i + 1 == n_steps)

    def join(self):
        """Order the current stream after every copy issued so far (the
        host buffers are complete once the current stream reaches here)."""
        main = torch.cuda.current_stream()
        main.wait_stream(self._d2h)
        main.wait_stream(self._h2d)

    def synchronize(self):
        self._d2h.synchronize()
        self._h2d.synchronize()
        torch.cuda.current_stream().synchronize()

    @property
    def bytes_per_member_step(self):
        """(host->device, device->host) bytes copied per member and step."""
        b = sum(self.host[0][a][sl].numel() * self.host[0][a].element_size() for a, sl in self._slices)
        return b, b


def _torch_dtype(grid):
    import numpy as np

    return torch.float64 if np.dtype(grid.dtype) == np.float64 else torch.float32
