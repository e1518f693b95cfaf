"""World-size-2 gloo tests (CPU) of the z-slab decomposition orchestration:
halo exchange directions, the all-to-all transposes of the spectral solve,
slab bookkeeping and the distributed RK4 step, against the single-process
oracle of the reference step."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stagflow_np as O

SHAPE = (8, 6, 4)
NU, DT, FORCE = 0.05, 0.01, (0.2, 0.0, -0.1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_case():
    bounds = [O.uniform_bounds(0.0, 1.0 + 0.3 * a, n) for a, n in enumerate(SHAPE)]
    g = O.OGrid(bounds, (True,) * 3)
    rng = np.random.default_rng(3)
    u = g.zeros_vel()
    for a in range(3):
        u[a][g.udof(a)] = rng.standard_normal(g.shape)
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    O.project_into(g, bcs, solve, u)
    return bounds, g, u


def _worker(rank, size, port, outdir, nsteps, defer=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        from _cpu_slab import CpuSlabBackend
        from paper_2604_18536_b200.distributed import Comm, SlabLayout, SlabSimulation, scatter_field

        bounds, g, u = _global_case()
        lay = SlabLayout(SHAPE[0], rank, size)
        be = CpuSlabBackend(bounds, lay, NU, FORCE)
        comm = Comm(lay)
        sim = SlabSimulation(be, comm)
        loc = be.new_field()
        for a, arr in enumerate(scatter_field(u, lay)):
            loc.u[a].copy_(torch.from_numpy(arr))
        st = sim.new_state(loc)
        if defer:
            sim.run_steps(st, nsteps, DT)
        else:
            for _ in range(nsteps):
                sim.rk4_step(st, DT)
        ke = sim.kinetic_energy(st.u)
        m = lay.m
        parts = [st.u.u[a][1:m + 1].contiguous() for a in range(3)] + [st.pressure.data[1:m + 1].contiguous()]
        gathered = []
        for t in parts:
            buf = [torch.empty_like(t) for _ in range(size)] if rank == 0 else None
            dist.gather(t, buf, dst=0)
            gathered.append(buf)
        # halo check: ghost plane 0 must equal the previous rank's last plane
        prev_last = torch.empty_like(st.u.u[0][m])
        nxt = (rank + 1) % size
        ops = [dist.P2POp(dist.isend, st.u.u[0][m].contiguous(), nxt), dist.P2POp(dist.irecv, prev_last, (rank - 1) % size)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        assert torch.equal(prev_last, st.u.u[0][0])
        if rank == 0:
            np.savez(os.path.join(outdir, "out.npz"), ke=ke,
                     **{f"f{i}": torch.cat(gathered[i], 0).numpy() for i in range(4)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nsteps,defer", [(1, False), (2, False), (3, True)])
def test_slab_rk4_world2_matches_oracle(nsteps, defer):
    """world 2 (gloo): rk4_step, and run_steps with each step's last
    projection deferred into the next step's stage 0 (u0_out)."""
    size = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(size, _free_port(), d, nsteps, defer), nprocs=size, join=True)
        z = np.load(os.path.join(d, "out.npz"))
        bounds, g, u = _global_case()
        bcs = O.periodic_bcs(3)
        solve = O.SpectralSolve(g)
        for _ in range(nsteps):
            u, p = O.rk_step(g, bcs, solve, u, DT, O.RK4, NU, FORCE)
        inner = tuple(slice(1, n + 1) for n in g.shape)
        for a in range(3):
            ref = u[a][inner]
            assert np.max(np.abs(z[f"f{a}"][:, 1:-1, 1:-1] - ref)) <= 1e-12 * np.max(np.abs(ref))
        refp = p[inner]
        assert np.max(np.abs(z["f3"][:, 1:-1, 1:-1] - refp)) <= 1e-11 * np.max(np.abs(refp))
        assert abs(float(z["ke"]) - O.kinetic_energy(g, u)) <= 1e-12 * O.kinetic_energy(g, u)


def test_slab_layout_and_tables():
    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200.distributed import SlabGrid, SlabLayout

    g = P.Grid([P.uniform_grid(0, 1, 8), P.uniform_grid(0, 1, 6), P.uniform_grid(0, 1, 4)], (True,) * 3)
    for rank in range(2):
        lay = SlabLayout(8, rank, 2)
        sg = SlabGrid(g, lay)
        assert sg.shape == (4, 6, 4) and list(lay.global_planes()) == list(range(rank * 4 + 1, rank * 4 + 5))
        pk, full = sg.packed_tables(), g.packed_tables()
        E0 = 10
        for t in range(10):
            np.testing.assert_array_equal(pk[t * 6:(t + 1) * 6], full[t * E0 + rank * 4: t * E0 + rank * 4 + 6])
        np.testing.assert_array_equal(pk[60:], full[100:])
    with pytest.raises(ValueError):
        SlabLayout(9, 0, 2)
