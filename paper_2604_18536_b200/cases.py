"""Initial conditions and canonical cases (mirror of cases.py:1-279, plus the
3D generators BASELINE.json's configs need but the reference lacks).

* ``taylor_green`` (2D, cases.py:33-54) and ``l2_error`` (cases.py:58-70).
* ``taylor_green_3d``: u = sin x cos y cos z, v = -cos x sin y cos z, w = 0
  sampled at the staggered points of [0, 2pi]^3 (discretely divergence-free
  on uniform grids).
* ``isotropic``: random-phase solenoidal field with E(k) ~ k^4 exp(-2 (k/k0)^2),
  unit-std components, made discretely divergence-free by the GPU projection.
* channel grid / IC / setup (cases.py:191-279).

These build inputs; they are not part of the timed path.
"""

import math

import numpy as np
import torch

from .bcs import BoundarySpec
from .errors import ConfigurationError
from .fields import ScalarField, VelocityField, fill_ghosts_scalar, fill_ghosts_velocity
from .grid import Grid, tanh_grid, uniform_grid
from .operators import velocity_weights
from .timestep import Setup

TWO_PI = 2.0 * math.pi


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _coord(grid, table, axis):
    shape = [1] * grid.dim
    shape[axis] = table.shape[0]
    return torch.from_numpy(np.array(table, dtype=np.float64)).to(_dev()).reshape(shape)


def taylor_green(grid, nu, t=0.0):
    """cases.py:33-54 (2D decaying vortex on [0, 2pi]^2)."""
    if grid.dim != 2:
        raise ConfigurationError("the vortex solution is two-dimensional")
    if not all(grid.periodic):
        raise ConfigurationError("the vortex solution requires periodic axes")
    for ax in grid.axes:
        if not (abs(ax.a) < 1e-12 and abs(ax.b - TWO_PI) < 1e-12):
            raise ConfigurationError("the vortex domain is [0, 2*pi]^2")
    decay = math.exp(-2.0 * nu * t)
    xf, yc = _coord(grid, grid.xb[0], 0), _coord(grid, grid.xc[1], 1)
    xc, yf = _coord(grid, grid.xc[0], 0), _coord(grid, grid.xb[1], 1)
    # evaluated on the host in float64 like the reference, then cast
    u = VelocityField(grid)
    ext = grid.ext_shape
    u.u[0].copy_((-torch.cos(xf) * torch.sin(yc) * decay).expand(ext))
    u.u[1].copy_((torch.sin(xc) * torch.cos(yf) * decay).expand(ext))
    p = ScalarField(grid)
    p.data.copy_((-0.25 * (torch.cos(2.0 * xc) + torch.cos(2.0 * yc)) * decay**2).expand(ext))
    bcs = BoundarySpec.all_periodic(2)
    fill_ghosts_velocity(u, bcs)
    fill_ghosts_scalar(p, bcs)
    return u, p


def taylor_green_grid(n, profile="uniform", gamma=1.5, dtype=np.float64):
    """cases.py:73-82"""
    if profile == "uniform":
        ax, ay = uniform_grid(0.0, TWO_PI, n), uniform_grid(0.0, TWO_PI, n)
    elif profile == "tanh":
        ax, ay = tanh_grid(0.0, TWO_PI, n, gamma), tanh_grid(0.0, TWO_PI, n, gamma)
    else:
        raise ConfigurationError(f"unknown study grid profile: {profile!r}")
    return Grid((ax, ay), (True, True), dtype=dtype)


def periodic_box(n, dtype=np.float64, length=TWO_PI):
    """Uniform triply periodic [0, L]^3 grid with n (int or 3-tuple) volumes."""
    ns = (n, n, n) if np.isscalar(n) else tuple(n)
    return Grid(tuple(uniform_grid(0.0, length, m) for m in ns), (True, True, True), dtype=dtype)


def taylor_green_3d(grid):
    """3D Taylor--Green vortex at the staggered points (w = 0)."""
    if grid.dim != 3:
        raise ConfigurationError("taylor_green_3d needs a 3D grid")
    ext = grid.ext_shape
    u = VelocityField(grid)
    x = [[_coord(grid, grid.face_coords(a)[g], g) for g in range(3)] for a in range(3)]
    u.u[0].copy_((torch.sin(x[0][0]) * torch.cos(x[0][1]) * torch.cos(x[0][2])).expand(ext))
    u.u[1].copy_((-torch.cos(x[1][0]) * torch.sin(x[1][1]) * torch.cos(x[1][2])).expand(ext))
    fill_ghosts_velocity(u, BoundarySpec.all_periodic(3))
    return u


def isotropic(grid, solver, seed=0, k0=4.0):
    """Random-phase solenoidal field, E(k) ~ k^4 exp(-2 (k/k0)^2), unit-std
    components, projected by the GPU spectral solver."""
    if grid.dim != 3 or not all(grid.periodic):
        raise ConfigurationError("isotropic IC needs a triply periodic 3D grid")
    dev = _dev()
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    n0, n1, n2 = grid.shape
    kx = torch.fft.fftfreq(n0, d=1.0 / n0, device=dev).reshape(-1, 1, 1)
    ky = torch.fft.fftfreq(n1, d=1.0 / n1, device=dev).reshape(1, -1, 1)
    kz = torch.fft.rfftfreq(n2, d=1.0 / n2, device=dev).reshape(1, 1, -1)
    kk = torch.sqrt(kx * kx + ky * ky + kz * kz)
    amp = torch.where(kk > 0, kk * torch.exp(-((kk / k0) ** 2)), torch.zeros_like(kk))  # sqrt(E/k^2) ~ k exp(-(k/k0)^2)
    u = VelocityField(grid)
    sl = grid.p_slices()
    tdt = u.u[0].dtype
    for a in range(3):
        noise = torch.randn((n0, n1, n2), generator=gen, device=dev, dtype=torch.float64)
        f = torch.fft.irfftn(torch.fft.rfftn(noise) * amp, s=(n0, n1, n2))
        f = f / f.std()
        u.u[a][sl] = f.to(tdt)
    bcs = BoundarySpec.all_periodic(3)
    fill_ghosts_velocity(u, bcs)
    from .poisson import project_into

    project_into(u, solver, bcs)
    return u


def l2_error(u_num, u_exact):
    """cases.py:58-70"""
    grid = u_num.grid
    if u_exact.grid.shape != grid.shape:
        raise ValueError("fields live on different grids")
    total = 0.0
    for a, w in enumerate(velocity_weights(grid)):
        sl = grid.u_slices(a)
        d = u_num.u[a][sl].double() - u_exact.u[a][sl].double()
        wt = torch.from_numpy(w.astype(np.float64)).to(d.device)
        total += float(torch.sum(wt * d * d).item())
    return math.sqrt(total)


def channel_grid(nx, ny, nz, gamma=2.0, y_profile="tanh", dtype=np.float64,
                 lx=4.0 * math.pi, ly=2.0, lz=4.0 * math.pi / 3.0):
    """cases.py:191-201"""
    ax = uniform_grid(0.0, lx, nx)
    if y_profile == "tanh":
        ay = tanh_grid(0.0, ly, ny, gamma)
    elif y_profile == "uniform":
        ay = uniform_grid(0.0, ly, ny)
    else:
        raise ConfigurationError(f"unknown wall-normal profile: {y_profile!r}")
    az = uniform_grid(0.0, lz, nz)
    return Grid((ax, ay, az), (True, False, True), dtype=dtype)


def channel_ic(grid, nu, force_x=1.0, perturbation=0.1, seed=0):
    """cases.py:204-237: laminar force balance + seeded sinusoidal wobble
    (same random draws, evaluated in float64 on the host, then uploaded)."""
    rng = np.random.default_rng(seed)
    lx = grid.axes[0].b - grid.axes[0].a
    ly = grid.axes[1].b - grid.axes[1].a
    lz = grid.axes[2].b - grid.axes[2].a
    scale = force_x / (2.0 * nu)
    u_tau_ref = math.sqrt(abs(force_x) * ly / 2.0)
    comps = []
    for a in range(3):
        fc = grid.face_coords(a)
        x = grid.broadcast(fc[0], 0)
        y = grid.broadcast(fc[1], 1)
        z = grid.broadcast(fc[2], 2)
        shape_y = y * (ly - y) * (4.0 / (ly * ly))
        base = scale * y * (ly - y) if a == 0 else 0.0
        wob = np.zeros(grid.ext_shape, dtype=grid.dtype)
        for _ in range(3):
            kx = rng.integers(1, 4)
            kz = rng.integers(1, 4)
            phx = rng.uniform(0, TWO_PI)
            phz = rng.uniform(0, TWO_PI)
            amp = rng.uniform(0.5, 1.0)
            wob += amp * np.sin(TWO_PI * kx * x / lx + phx) * np.sin(TWO_PI * kz * z / lz + phz)
        arr = np.empty(grid.ext_shape, dtype=grid.dtype)
        arr[...] = base + perturbation * u_tau_ref * shape_y * wob
        comps.append(arr)
    return VelocityField(grid, comps)


def channel_setup(nx, ny, nz, gamma=2.0, nu=1.0 / 180.0, force=(1.0, 0.0, 0.0), y_profile="tanh",
                  dtype=np.float64, solver="direct", method="ssp33", closure=None, seed=0, perturbation=0.1,
                  cfl_conv=0.85, cfl_diff=0.85, dt_max=0.05):
    """cases.py:240-274"""
    grid = channel_grid(nx, ny, nz, gamma=gamma, y_profile=y_profile, dtype=dtype)
    bcs = BoundarySpec.channel(dim=3, wall_axis=1)
    return Setup(grid, bcs, nu=nu, force=force, closure=closure, solver=solver, method=method,
                 cfl_conv=cfl_conv, cfl_diff=cfl_diff, dt_max=dt_max,
                 ic=lambda g: channel_ic(g, nu, force_x=force[0], perturbation=perturbation, seed=seed))


def poiseuille_profile(y, force_x, nu, ly=2.0):
    """cases.py:277-279"""
    return force_x * y * (ly - y) / (2.0 * nu)
