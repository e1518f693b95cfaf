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


# ---------------------------------------------------------------------------
# file formats (stats.py:170-228, csvio.py:1-31): the reference's byte layout,
# so profiles and snapshots written here are read by stagflow and vice versa
# ---------------------------------------------------------------------------
def _atomic_write(path, data, mode):
    import os
    import tempfile

    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-")
    try:
        with os.fdopen(fd, mode) as fh:
            if callable(data):
                data(fh)
            else:
                fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def write_profile_csv(path, profile):
    """stats.py:170-178 + csvio.write_csv: schema comment, header, full-
    precision floats, one row per wall-normal point."""
    names = profile.column_names()
    lines = ["# stagflow-csv v1 stat-profile", ",".join(names)]
    for r in profile.rows():
        lines.append(",".join(repr(float(v)) for v in r))
    _atomic_write(str(path), "\n".join(lines) + "\n", "w")


def _host_components(u):
    comps = []
    for c in u.u:
        a = c.detach().cpu().numpy() if hasattr(c, "detach") else np.asarray(c)
        comps.append(np.ascontiguousarray(a, dtype=a.dtype.newbyteorder("<")))
    return comps


def write_snapshot(path_base, u, t):
    """stats.py:181-211: raw little-endian dump of the extended components
    plus a text sidecar (time, dtype, components, shapes), both atomic."""
    comps = _host_components(u)

    def dump(fh):
        for c in comps:
            c.tofile(fh)

    _atomic_write(str(path_base) + ".bin", dump, "wb")
    lines = [f"time {t!r}", f"dtype {comps[0].dtype.name}", f"components {len(comps)}"]
    for i, c in enumerate(comps):
        lines.append(f"shape{i} " + " ".join(str(n) for n in c.shape))
    _atomic_write(str(path_base) + ".txt", "\n".join(lines) + "\n", "w")


def read_snapshot(path_base):
    """stats.py:214-228: inverse of write_snapshot; returns (arrays, time)."""
    meta = {}
    with open(str(path_base) + ".txt") as fh:
        for line in fh:
            key, _, rest = line.strip().partition(" ")
            meta[key] = rest
    dtype = np.dtype(meta["dtype"]).newbyteorder("<")
    n = int(meta["components"])
    shapes = [tuple(int(v) for v in meta[f"shape{i}"].split()) for i in range(n)]
    arrays = []
    with open(str(path_base) + ".bin", "rb") as fh:
        for shape in shapes:
            arrays.append(np.fromfile(fh, dtype=dtype, count=int(np.prod(shape))).reshape(shape))
    return arrays, float(meta["time"])
