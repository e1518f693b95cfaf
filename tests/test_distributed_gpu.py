"""GPU tests of the z-slab path with the CUDA backend (C ABI sfb_slab_*):
P = 1 on one GPU, and P = 2 as two processes sharing cuda:0 with gloo and
host-staged communication (this environment exposes a single GPU; NCCL needs
one GPU per rank)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stagflow_np as O

pytestmark = pytest.mark.gpu

SHAPE = (16, 12, 10)
NU, DT, FORCE = 0.02, 5e-3, (0.1, 0.0, 0.0)


def _case():
    bounds = [O.uniform_bounds(0.0, 1.0 + 0.3 * a, n) for a, n in enumerate(SHAPE)]
    g = O.OGrid(bounds, (True,) * 3)
    rng = np.random.default_rng(11)
    u = g.zeros_vel()
    for a in range(3):
        u[a][g.udof(a)] = rng.standard_normal(g.shape)
    O.project_into(g, O.periodic_bcs(3), O.SpectralSolve(g), u)
    return bounds, g, u


def _run(rank, size, stage_host, nsteps, nccl=False, defer=False):
    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200.distributed import (Comm, CudaSlabBackend, NcclComm, SlabGrid, SlabLayout,
                                                   SlabSimulation, scatter_field)

    bounds, g, u = _case()
    pg = P.Grid(tuple(P.AxisCoords(b) for b in bounds), (True,) * 3)
    lay = SlabLayout(SHAPE[0], rank, size)
    sg = SlabGrid(pg, lay)
    be = CudaSlabBackend(sg, NU, FORCE)
    sim = SlabSimulation(be, NcclComm(lay) if nccl else Comm(lay, stage_host=stage_host))
    loc = be.new_field()
    for a, arr in enumerate(scatter_field(u, lay)):
        loc.u[a].copy_(torch.from_numpy(arr))
    st = sim.new_state(loc)
    if defer:
        sim.run_steps(st, nsteps, DT)
    else:
        for _ in range(nsteps):
            sim.rk4_step(st, DT)
    torch.cuda.synchronize()
    m = lay.m
    return [st.u.u[a][1:m + 1].cpu() for a in range(3)] + [st.pressure.data[1:m + 1].cpu()], sim.kinetic_energy(st.u)


def _check(fields, ke, nsteps):
    bounds, g, u = _case()
    solve = O.SpectralSolve(g)
    for _ in range(nsteps):
        u, p = O.rk_step(g, O.periodic_bcs(3), solve, u, DT, O.RK4, NU, FORCE)
    inner = tuple(slice(1, n + 1) for n in g.shape)
    for a in range(3):
        ref = u[a][inner]
        got = fields[a][:, 1:-1, 1:-1]
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), a
    refp = p[inner]
    assert np.max(np.abs(fields[3][:, 1:-1, 1:-1] - refp)) <= 1e-12 * np.max(np.abs(refp))
    assert abs(ke - O.kinetic_energy(g, u)) <= 1e-12 * O.kinetic_energy(g, u)


def test_slab_p1_cuda_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    fields, ke = _run(0, 1, False, 2)
    _check([f.numpy() for f in fields], ke, 2)


def test_slab_p1_nccl_comm_matches_oracle():
    """The same two RK4 steps through the library's own NCCL communicator
    (sfb_comm_*: one-rank communicator, halo / all-to-all / all-reduce
    through the C ABI)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    fields, ke = _run(0, 1, False, 2, nccl=True)
    _check([f.numpy() for f in fields], ke, 2)


def test_slab_p1_run_steps_deferred_matches_oracle():
    """run_steps on the slab (NCCL communicator): each step's last projection
    applied by the next step's stage 0 (FL_U0P on the halo plan)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    fields, ke = _run(0, 1, False, 3, nccl=True, defer=True)
    _check([f.numpy() for f in fields], ke, 3)


def test_nccl_comm_ops_one_rank():
    """sfb_comm_* at one rank: periodic self halo, all-to-all and
    send/recv as device copies on the caller's stream, all-reduce identity."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2604_18536_b200.distributed import NcclComm, SlabLayout

    c = NcclComm(SlabLayout(4, 0, 1))
    f = [torch.randn(6, 5, 7, dtype=torch.float64, device="cuda") for _ in range(3)]
    ref = [x.clone() for x in f]
    c.halo(f)
    for x, r in zip(f, ref):
        assert torch.equal(x[0], r[4]) and torch.equal(x[5], r[1]) and torch.equal(x[1:5], r[1:5])
    a = torch.randn(1000, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    c.all_to_all_async(b, a).wait()
    assert torch.equal(a, b)
    p, q = torch.randn(33, device="cuda"), torch.zeros(33, device="cuda")
    c.plane_from_next(p, q)
    assert torch.equal(p, q)
    t = torch.tensor([2.5, -1.0], dtype=torch.float64, device="cuda")
    assert torch.equal(c.allreduce_device(t.clone(), "min"), t)
    assert c.allreduce(3.25) == 3.25


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, size, port, outdir, defer=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        fields, ke = _run(rank, size, True, 2, defer=defer)
        gathered = []
        for t in fields:
            t = t.contiguous()
            buf = [torch.empty_like(t) for _ in range(size)] if rank == 0 else None
            dist.gather(t, buf, dst=0)
            gathered.append(buf)
        if rank == 0:
            np.savez(os.path.join(outdir, "out.npz"), ke=ke,
                     **{f"f{i}": torch.cat(gathered[i], 0).numpy() for i in range(4)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("defer", [False, True])
def test_slab_p2_cuda_two_processes_matches_oracle(defer):
    """P = 2 on one device (host-staged gloo): rk4_step, and run_steps with
    the deferred last projection (stage 0 reads the exchanged unprojected
    ghost planes and the neighbours' pressure planes)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, defer), nprocs=2, join=True)
        z = np.load(os.path.join(d, "out.npz"))
        _check([z[f"f{i}"] for i in range(4)], float(z["ke"]), 2)
