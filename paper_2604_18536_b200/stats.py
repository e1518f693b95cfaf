"""Plane-averaged turbulence statistics for wall-bounded flows on the GPU
(mirror of stats.py:17-167).  The per-snapshot plane reductions run on the
device (csrc/stats.cu): the snapshot is never copied to the host; only one
row of sums per wall-normal index comes back.  The snapshot average is taken
in long double like the reference (stats.py:126-130)."""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError
from .fields import fill_ghosts_velocity
from .operators import _plan
from .plan import stream_ptr
from .poisson import homogeneous


@dataclass
class StatProfile:
    """One row per wall-normal volume; see ``column_names`` for layout."""

    y: np.ndarray
    y_plus: np.ndarray
    u_mean: np.ndarray
    rms: np.ndarray
    u3: np.ndarray
    u4: np.ndarray
    uuv: np.ndarray
    uw: np.ndarray
    nut_over_nu: np.ndarray
    u_tau: float
    n_snapshots: int

    def column_names(self):
        d = self.u_mean.shape[0]
        names = ["y", "y_plus"]
        names += [f"u{c}_mean" for c in range(d)]
        names += [f"u{c}_rms" for c in range(d)]
        names += ["u0_3rd", "u0_4th", "uuv", "uw", "nut_over_nu"]
        return names

    def rows(self):
        cols = [self.y, self.y_plus]
        cols += list(self.u_mean)
        cols += list(self.rms)
        cols += [self.u3, self.u4, self.uuv, self.uw, self.nut_over_nu]
        return np.stack(cols, axis=1)


def _plane_sums(grid, wall_axis, comps, mode):
    nj = grid.shape[wall_axis]
    nq = grid.dim if mode == 0 else 7
    out = torch.empty(nq * nj, dtype=torch.float64, device="cuda")
    N.call("sfb_plane_sums", _plan(grid), int(wall_axis), N.ptr3(comps), int(mode), ctypes.c_void_p(out.data_ptr()),
           stream_ptr())
    return out


def _tmean(parts):
    acc = np.sum(np.stack(parts).astype(np.longdouble), axis=0)
    return (acc / len(parts)).astype(np.float64)


def accumulate_stats(snapshots, bcs, nu, wall_axis=1, nut_snapshots=None):
    """stats.py:55-167: reduce velocity snapshots (two homogeneous periodic
    directions) to a wall-normal statistics profile."""
    snapshots = list(snapshots)
    if len(snapshots) < 2:
        raise ValueError("need at least two snapshots to average")
    grid = snapshots[0].grid
    d = grid.dim
    if wall_axis != 1:
        raise ConfigurationError("GPU statistics support the wall-normal axis 1 (the channel layout)")
    ny = grid.shape[wall_axis]
    plane = int(np.prod([n for a, n in enumerate(grid.shape) if a != wall_axis]))
    hom = homogeneous(bcs)
    per = {k: [] for k in ("mean", "rms", "u3", "u4", "uuv", "uw")}
    for snap in snapshots:
        up = snap.copy()
        fill_ghosts_velocity(up, bcs)
        sums = _plane_sums(grid, wall_axis, up.u, 0)
        full_mean = sums / plane  # (d, ny) plane means at every interior wall index
        means = full_mean.view(d, ny).cpu().numpy().astype(np.float64)
        N.call("sfb_sub_plane_mean", _plan(grid), int(wall_axis), N.ptr3(up.u), ctypes.c_void_p(full_mean.data_ptr()),
               stream_ptr())
        fill_ghosts_velocity(up, hom)
        mom = (_plane_sums(grid, wall_axis, up.u, 1) / plane).view(7, ny).cpu().numpy()
        mean_profile = np.zeros((d, ny))
        rms_profile = np.zeros((d, ny))
        other = 2 if wall_axis != 2 else 1
        for a in range(d):
            if a == wall_axis:
                if grid.periodic[a]:
                    mean_profile[a] = means[a]
                else:
                    face = means[a][: ny - 1]  # DOF faces 1..ny-1 (stats.py:97-102)
                    mean_profile[a] = 0.5 * (np.concatenate(([0.0], face)) + np.concatenate((face, [0.0])))
                rms_profile[a] = np.sqrt(mom[2])
            else:
                mean_profile[a] = means[a]
                rms_profile[a] = np.sqrt(mom[0] if a == 0 else mom[1] if a == other else mom[0])
        per["mean"].append(mean_profile)
        per["rms"].append(rms_profile)
        per["u3"].append(mom[3])
        per["u4"].append(mom[4])
        per["uuv"].append(mom[5])
        per["uw"].append(mom[6])
    u_mean = _tmean(per["mean"])
    if nut_snapshots:
        prof = []
        for f in nut_snapshots:
            s = _plane_sums(grid, wall_axis, [f.data] * d, 0)
            prof.append((s / plane).view(d, ny)[0].cpu().numpy())
        nut_over_nu = _tmean(prof) / nu
    else:
        nut_over_nu = np.zeros(ny)
    y = np.asarray(grid.axes[wall_axis].centers, dtype=np.float64)
    du_dy = u_mean[0][0] / y[0]
    u_tau = float(np.sqrt(nu * max(du_dy, 0.0)))
    return StatProfile(y=y, y_plus=y / nu, u_mean=u_mean, rms=_tmean(per["rms"]), u3=_tmean(per["u3"]),
                       u4=_tmean(per["u4"]), uuv=_tmean(per["uuv"]), uw=_tmean(per["uw"]), nut_over_nu=nut_over_nu,
                       u_tau=u_tau, n_snapshots=len(snapshots))
