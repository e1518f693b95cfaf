"""Benchmark: fp64 cell-updates/s per RK4 step (BASELINE.json metric).

Our arm (default):  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 840]
Reference arm:      python bench.py --impl reference [...]

A "step" is one projected RK4 step (4 fused RHS/stage launches, 4 spectral
projections) of the periodic DNS on the full grid resident in HBM; the K
timed steps are one ``run_steps(setup, K, dt)`` call (the reference's
fixed-step loop), which returns a fully projected state.  At N=1
the workload is BASELINE config 5, 840^3 fp64 on one B200 (the largest
single-GPU configuration; the metric is quoted at 512^3/840^3), started from
a seeded random-phase isotropic field (synthetic data).  Every field is
4.7 GB, far larger than the 126 MB L2, so no L2 flush is needed between
steps.  For N>1 each rank steps its own 840^3 slab replica of a
840 x 840 x 840N domain share (weak scaling).

The JSON line carries: value (device-timed, max over ranks), e2e (the same
metric through the public API with host buffers and H2D/D2H copies inside
the timed region), roofline of the dominant kernel (fused RK stage: algorithmic
bytes / CUDA-event time of its launches inside the timed region, vs the
measured HBM copy peak), cpu_baseline (the CPU oracle port of the reference
RK4 step on a bounded 128^3 sample), clocks sampled during the timed region,
and gpu_launches (our kernel launches in the timed region).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# stdout carries exactly one JSON line: NCCL's banner / info lines (printed to
# stdout when the environment sets NCCL_DEBUG=VERSION or INFO) go to stderr
os.environ["NCCL_DEBUG"] = "WARN"
os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
sys.path.insert(0, ROOT)

RK4_BYTES_PER_CELL_F64 = 864


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(n=128, steps=2):
    """The oracle port of the reference RK4 step (numpy/scipy, as stagflow
    runs it: ufuncs single-threaded, scipy.fft default 1 worker) on a bounded
    n^3 sample of the same workload."""
    import numpy as np

    from oracle import stagflow_np as O

    b = O.uniform_bounds(0.0, 2 * np.pi, n)
    g = O.OGrid([b, b, b], (True,) * 3)
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    rng = np.random.default_rng(0)
    u = g.zeros_vel()
    for a in range(3):
        u[a][g.udof(a)] = rng.standard_normal(g.shape)
    O.fill_velocity(g, bcs, u)
    O.project_into(g, bcs, solve, u)
    u, _ = O.rk_step(g, bcs, solve, u, 1e-3, O.RK4, 1 / 1600)  # warm-up
    t0 = time.perf_counter()
    c0 = time.process_time()
    for _ in range(steps):
        u, _ = O.rk_step(g, bcs, solve, u, 1e-3, O.RK4, 1 / 1600)
    wall = time.perf_counter() - t0
    cpu = time.process_time() - c0
    return {"value": n**3 * steps / wall, "unit": "cell-updates/s", "cores": 1, "kind": "port",
            "sample": f"{steps} RK4 steps of a {n}^3 fp64 periodic field (oracle port of stagflow rk_step, "
                      f"numpy+scipy.fft, 1 thread; {cpu / wall:.2f} cores busy on average)",
            "wall_s": wall}


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port) on the host,
    with every host thread it can use: numpy's ufuncs are single-threaded (as
    in stagflow), the FFTs of the pressure solve run on all cores
    (scipy.fft workers = cpu_count)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import contextlib

    import numpy as np

    try:
        import scipy.fft as sfft

        threads = os.cpu_count() or 1
        workers = sfft.set_workers(threads)
    except ImportError:  # numpy.fft fallback: single-threaded
        threads = 1
        workers = contextlib.nullcontext()

    from oracle import stagflow_np as O

    n = args.ref_n
    b = O.uniform_bounds(0.0, 2 * np.pi, n)
    g = O.OGrid([b, b, b], (True,) * 3)
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    rng = np.random.default_rng(0)
    u = g.zeros_vel()
    for a in range(3):
        u[a][g.udof(a)] = rng.standard_normal(g.shape)
    O.fill_velocity(g, bcs, u)
    O.project_into(g, bcs, solve, u)
    with workers:
        for _ in range(args.warmup):
            u, _ = O.rk_step(g, bcs, solve, u, 1e-3, O.RK4, 1 / 1600)
        t0 = time.perf_counter()
        c0 = time.process_time()
        for _ in range(args.steps):
            u, _ = O.rk_step(g, bcs, solve, u, 1e-3, O.RK4, 1 / 1600)
        wall = time.perf_counter() - t0
        cpu = time.process_time() - c0
    v = n**3 * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "cell-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"periodic DNS RK4 step, bounded {n}^3 sample of the {args.n}^3 config",
                   "method": "rk4", "solver": "spectral"},
        "cpu_baseline": {"value": v, "unit": "cell-updates/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} RK4 steps of a {n}^3 fp64 field (oracle port, numpy ufuncs + "
                                   f"scipy.fft on {threads} workers; {cpu / wall:.2f} cores busy on average)"},
        "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "fp64 cell-updates/s per RK4 step"


WEAK_LADDER = {1: (840, 840, 840), 2: (1680, 840, 840), 4: (1680, 1680, 840), 8: (1680, 1680, 1680)}


def _slab_tgv(local_grid, P):
    """3D Taylor-Green vortex at the local slab's staggered points (ghosts
    included; the domain is [0, 2 pi * n / n_ref] so the field is periodic)."""
    import torch

    u = P.VelocityField(local_grid)
    dev = u.u[0].device

    def c(tab, axis):
        shp = [1, 1, 1]
        shp[axis] = tab.shape[0]
        return torch.from_numpy(tab.astype("float64")).to(dev).reshape(shp)

    fc = [[c(local_grid.face_coords(a)[g], g) for g in range(3)] for a in range(3)]
    ext = local_grid.ext_shape
    u.u[0].copy_((torch.sin(fc[0][0]) * torch.cos(fc[0][1]) * torch.cos(fc[0][2])).expand(ext))
    u.u[1].copy_((-torch.cos(fc[1][0]) * torch.sin(fc[1][1]) * torch.cos(fc[1][2])).expand(ext))
    return u


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import _native as N
    from paper_2604_18536_b200 import cases
    from paper_2604_18536_b200 import timestep as TS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    dtype = np.float64 if args.dtype == "f64" else np.float32
    dt = 1e-3
    slab = world > 1 or args.slab
    if not slab:
        n = args.n
        gshape = (n, n, n)
        grid = cases.periodic_box(n, dtype=dtype)
        bcs = P.BoundarySpec.all_periodic(3)
        setup = P.Setup(grid, bcs, nu=1 / 1600, solver="spectral", method="rk4")
        u0 = cases.isotropic(grid, setup.solver, seed=rank)
        state = setup.new_state(u0=u0)
        del u0
        local_cells = n**3

        def step():
            P.rk_step(state, dt, P.RK4, setup.solver, setup)

        def steps(k):
            # the reference's fixed-step loop (timestep.py:317-337): each
            # step's last projection is finished by the next step's first
            # stage kernel; the state it returns is fully projected
            P.run_steps(setup, k, dt=dt, state=state, project_initial=False)

        def cur_u():
            return state.u

        def ke():
            return P.kinetic_energy(state.u)

        ic = "isotropic random-phase IC"
    else:
        from paper_2604_18536_b200.distributed import CudaSlabBackend, SlabGrid, SlabLayout, SlabSimulation, make_comm

        gshape = WEAK_LADDER.get(world) if args.n == 840 else (args.n * world, args.n, args.n)
        if gshape is None:
            gshape = (840 * world, 840, 840)
        ref = 840 if args.n == 840 else args.n
        gg = P.Grid(tuple(P.uniform_grid(0.0, 2 * np.pi * m / ref, m) for m in gshape), (True,) * 3, dtype=dtype)
        lay = SlabLayout(gshape[0], rank, world)
        sg = SlabGrid(gg, lay)
        be = CudaSlabBackend(sg, 1 / 1600, None)
        sim = SlabSimulation(be, make_comm(lay, group=dist.group.WORLD if world > 1 else None))
        st = sim.new_state(_slab_tgv(sg, P))
        sim.proj.project(st.u)
        local_cells = lay.m * gshape[1] * gshape[2]

        def step():
            sim.rk4_step(st, dt)

        def steps(k):
            # run_steps on the slab: each step's last projection is finished
            # by the next step's stage 0
            sim.run_steps(st, k, dt)

        def cur_u():
            return st.u

        def ke():
            return sim.kinetic_energy(st.u)

        ic = "3D Taylor-Green IC"
    steps(args.warmup)
    torch.cuda.synchronize()
    barrier()

    # ---- device-timed region
    TS.STAGE_EVENTS = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = N.launches
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        start.record()
        steps(args.steps)
        end.record()
        torch.cuda.synchronize()
    launches = N.launches - launches0
    ms = start.elapsed_time(end) / args.steps
    ev = TS.STAGE_EVENTS
    TS.STAGE_EVENTS = None
    st_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in ev)
    st_bytes = sum(bpc for _, _, bpc in ev) * local_cells
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_cells = int(np.prod(gshape))
    value = total_cells / (ms_max * 1e-3)

    # ---- end to end through the public API with pinned host buffers
    u = cur_u()
    ext = u.u[0].shape
    host = [torch.empty(ext, dtype=u.u[0].dtype, pin_memory=True) for _ in range(3)]
    for a in range(3):
        host[a].copy_(u.u[a])
    torch.cuda.synchronize()
    barrier()
    # the e2e leg has its own step count: its first uploads are not
    # overlapped, so a few more steps than the device-timed leg
    e2e_steps = max(1, args.e2e_steps)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    ens_info = None
    if not slab and not args.e2e_serial:
        # HostEnsemble (the package's host-memory stepping API): two
        # independent trajectories in pinned host memory -- the bench state
        # and a copy translated by n/2 planes along axis 0 (an exact symmetry
        # of the periodic uniform box, so a different but equally valid
        # state).  Every member step uploads its velocity, steps, reads it
        # back; one member's copies overlap the other member's step.
        host2 = [torch.empty(ext, dtype=u.u[0].dtype, pin_memory=True) for _ in range(3)]
        for a in range(3):
            host2[a].copy_(host[a])
            host2[a][1:-1].copy_(torch.roll(host[a][1:-1], gshape[0] // 2, dims=0))
        ens = P.HostEnsemble(setup, [host, host2], chunks=8, state=state)
        rounds = max(1, e2e_steps // 2)
        torch.cuda.synchronize()
        es.record()
        ens.run(rounds, dt)
        ens.join()
        ee.record()
        torch.cuda.synchronize()
        e2e_steps = 2 * rounds
        e2e_ms = es.elapsed_time(ee) / e2e_steps
        ens_info = {"members": 2, "rounds": rounds}
        del ens, host2
        # the chained single-trajectory figure beside it (every step waits for
        # its own upload; read-back and re-upload overlap chunk by chunk)
        ser_steps = max(1, min(3, e2e_steps))
    else:
        ser_steps = e2e_steps
    # each step: the pinned host velocity goes in, the step runs, the result
    # comes back.  The copies run on the two copy engines in chunks of planes
    # (PCIe is full duplex): the upload of chunk c for the next step waits
    # only for chunk c's read-back, so the read-back and the re-upload
    # overlap chunk by chunk
    d2h_s, h2d_s = torch.cuda.Stream(), torch.cuda.Stream()
    nchunk = 8
    bounds = [round(c * ext[0] / nchunk) for c in range(nchunk + 1)]
    chunks = [(a, slice(bounds[c], bounds[c + 1])) for a in range(3) for c in range(nchunk)]
    evs = [torch.cuda.Event() for _ in chunks]
    torch.cuda.synchronize()
    es.record()
    u = cur_u()
    for a in range(3):
        u.u[a].copy_(host[a], non_blocking=True)
    for it in range(ser_steps):
        step()
        u = cur_u()
        d2h_s.wait_stream(main)
        last = it == ser_steps - 1
        with torch.cuda.stream(d2h_s):
            for (a, sl), ev in zip(chunks, evs):
                host[a][sl].copy_(u.u[a][sl], non_blocking=True)
                ev.record(d2h_s)
        if not last:
            with torch.cuda.stream(h2d_s):
                for (a, sl), ev in zip(chunks, evs):
                    h2d_s.wait_event(ev)
                    u.u[a][sl].copy_(host[a][sl], non_blocking=True)
        main.wait_stream(d2h_s)
        main.wait_stream(h2d_s)
    ee.record()
    torch.cuda.synchronize()
    ser_ms = es.elapsed_time(ee) / ser_steps
    if ens_info is None:
        e2e_ms = ser_ms
    t = torch.tensor([e2e_ms, ser_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms, ser_ms = (float(x) for x in t.tolist())
    field_bytes = int(np.prod(ext)) * np.dtype(dtype).itemsize
    ke_after = ke()
    # device memory in use per rank (cudaMemGetInfo), max over ranks
    free_b, total_b = torch.cuda.mem_get_info()
    mem = torch.tensor([float(total_b - free_b)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(mem, op=dist.ReduceOp.MAX)
    hbm_used_gb = float(mem.item()) / 1e9

    # other BASELINE configs, measured on the same box by the same run (rank 0
    # at N=1): the 840^3 fields are released first
    others = []
    if world == 1 and not slab and not args.no_extras:
        del u, host
        state = setup = None  # noqa: F841 (release the 840^3 registers)
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        others = run_other_configs()

    if rank == 0:
        peak, peak_kind = _peaks()
        achieved = st_bytes / (st_ms * 1e-3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("stage_kernel", {}).get("dram_bytes_per_launch")
            except (ValueError, OSError):
                traffic = None
        bpc = RK4_BYTES_PER_CELL_F64 * (np.dtype(dtype).itemsize / 8)
        step_gbs = bpc * local_cells / (ms * 1e-3) / 1e9
        wl = (f"periodic DNS {gshape[0]}x{gshape[1]}x{gshape[2]} {args.dtype} RK4 step, "
              + ("BASELINE config 5 (840^3 on one B200)" if world == 1 and not slab else
                 f"z-slab decomposed over {world} GPU(s), {lay.m} planes per rank (weak ladder, SURVEY 7)")
              + f", {ic}, spectral projection")
        line = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": wl, "grid": list(gshape), "method": "rk4", "solver": "spectral",
                       "nu": 1 / 1600, "dt": dt,
                       "l2": "inputs larger than L2 (each field >= 4.7 GB at 840^3 per GPU); no flush needed",
                       "parallelism": f"z-slab x{world}" if slab else "single GPU",
                       **({"comm": type(sim.comm).__name__} if slab else {})},
            "e2e": {"value": total_cells / (e2e_ms * 1e-3), "unit": "cell-updates/s",
                    "h2d_bytes_per_step": 3 * field_bytes * world, "d2h_bytes_per_step": 3 * field_bytes * world,
                    "steps": e2e_steps,
                    "api": (("HostEnsemble.run: 2 independent trajectories in pinned host memory, every member step "
                             "uploads the member's velocity, runs rk_step and reads it back (24 plane chunks on the "
                             "two copy engines); one member's copies overlap the other member's step"
                             if ens_info else
                             "rk_step (or the slab stepper) with pinned host velocity copied in and out every step; "
                             "copies in 24 plane chunks on the two copy engines, each chunk's re-upload "
                             "ordered after its own read-back")),
                    **({"ensemble": ens_info} if ens_info else {}),
                    "serial": {"value": total_cells / (ser_ms * 1e-3), "steps": ser_steps,
                               "api": "one trajectory: upload -> rk_step -> read back, each step waiting for its "
                                      "own upload"}},
            "roofline": {"bound": "hbm", "kernel": "k_stage_march (fused RHS + RK stage combine)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_kind": peak_kind, "traffic": traffic,
                         "bytes_per_cell": ("104 (72 on the first step)/128/128/80 B fp64 per stage launch: y, u0, s, y_next (and the written projected u0) fields "
                                            "+ the pressure on the stages that apply the previous projection"),
                         "stage_share_of_step": st_ms / (ms * args.steps)},
            "step_roofline": {"algorithmic_bytes_per_cell": bpc, "achieved": step_gbs, "peak": peak,
                              "frac": step_gbs / peak},
            "gpu_launches": launches,
            "hbm_gb": {"used_max_over_ranks": hbm_used_gb, "total_per_gpu": total_b / 1e9},
            "clocks": clocks.summary(),
            "ke_after": ke_after,
        }
        if others:
            line["other_configs"] = others
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_other_configs():
    """BASELINE configs 3-4 next to the headline (bench_extra.py cases, CUDA
    events, median of 5 after 2 warm-ups): 512^3 RK4 step fp64 and fp32, the
    512^3 RK4 unrolled gradient (tape + reverse sweep), the Re_tau=180
    channel 512x256x256 RK4 step.  A failing case reports its error."""
    import gc

    import torch

    import bench_extra as BE

    out = []
    for name, fn in (("step512", lambda: BE.case_step(512, "f64")), ("step512f32", lambda: BE.case_step(512, "f32")),
                     ("vjp512", lambda: BE.case_vjp(512)), ("channel", BE.case_channel)):
        try:
            out.append(fn())
        except Exception as exc:  # noqa: BLE001 - reported, the headline line still prints
            out.append({"case": name, "error": f"{type(exc).__name__}: {exc}"[:200]})
        gc.collect()
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=840)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--ref-n", type=int, default=96)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e from one chained trajectory only (no HostEnsemble)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other BASELINE configs (other_configs)")
    ap.add_argument("--slab", action="store_true", help="use the z-slab path even at N=1")
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # not under torchrun: launch one rank per GPU ourselves (same contract
        # as the driver's torch.distributed.run launch)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
