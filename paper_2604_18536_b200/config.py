"""Run configuration of the batch studies (config.py:1-261 of the reference),
extended with the keys the B200 path adds:

* ``run.device``   -- the CUDA device a run uses (``cuda``, ``cuda:N``);
* ``solver.kind``  -- also ``fft-tridiag`` (the channel's exact FFT x
  tridiagonal solver, ``ChannelPoissonSolver``);
* ``time.method``  -- also ``rk4``.

Same INI dialect and contract as the reference: sections and keys are
strict (an unknown one is a ``ConfigurationError`` naming the key and its
line), every key has a default except ``run.study``, enumerations and the
cross-field rules are checked, and ``emit_config`` writes the effective
configuration so that re-parsing it reproduces the same ``RunConfig``.
``build_setup`` is the reference's cli.build_setup (cli.py:76-110) on the
device path.
"""

import configparser
import io
import math

import numpy as np

from .errors import ConfigurationError

STUDIES = ("simulate", "convergence", "vcurve", "adjoint-check", "channel-smoke")


def _dt(text):
    return "adaptive" if text == "adaptive" else float(text)


def _floats(text):
    return tuple(float(v) for v in text.replace(",", " ").split())


def _ints(text):
    return tuple(int(v) for v in text.replace(",", " ").split())


def _axis_keys(ax):
    return [(f"{ax}_kind", str, "uniform"), (f"{ax}_a", float, 0.0), (f"{ax}_b", float, 2.0 * math.pi),
            (f"{ax}_n", int, 32), (f"{ax}_gamma", float, 1.5), (f"{ax}_s", float, 1.3)]


# (section, [(key, parser, default)]); default None = required.  Key order is
# the emitted order.
_LAYOUT = [
    ("run", [("study", str, None), ("precision", str, "f64"), ("seed", int, 0), ("outdir", str, "out"),
             ("threads", int, 0), ("observer_cadence", int, 10), ("write_snapshots", int, 0),
             ("device", str, "cuda")]),
    ("grid", [("dim", int, 2)] + _axis_keys("x") + _axis_keys("y") + _axis_keys("z")),
    ("bc", [("x", str, "periodic"), ("y", str, "periodic"), ("z", str, "periodic"),
            ("dirichlet_value", str, "zero"), ("constant_u", _floats, (0.0, 0.0, 0.0))]),
    ("physics", [("nu", float, 1e-3), ("force", str, "none"), ("force_vector", _floats, (1.0, 0.0, 0.0)),
                 ("closure", str, "none"), ("closure_c", float, -1.0), ("closure_p", float, -2.5),
                 ("closure_filter", str, "geometric")]),
    ("solver", [("kind", str, "direct"), ("tol", float, -1.0), ("max_iter", int, 0)]),
    ("time", [("method", str, "ssp33"), ("dt", _dt, "adaptive"), ("cfl_conv", float, 0.85),
              ("cfl_diff", float, 0.85), ("dt_max", float, 0.05), ("t_final", float, 1.0)]),
    ("study", [("convergence_ns", _ints, (16, 32, 64)), ("profile", str, "uniform"), ("gamma", float, 1.5),
               ("check_dt", int, 0), ("vcurve_decades", _floats, (-12.0, 0.0)), ("vcurve_points", int, 193),
               ("channel_n", _ints, (32, 48, 16)), ("channel_gamma", float, 2.0), ("channel_steps", int, 500),
               ("adjoint_seeds", int, 50)]),
]
SCHEMA = {sec: {k: (conv, dflt) for k, conv, dflt in keys} for sec, keys in _LAYOUT}

_PROFILES = ("uniform", "cosine", "tanh", "stretched")
_BCS = ("periodic", "dirichlet", "symmetric")
CHOICES = {
    ("run", "study"): STUDIES,
    ("run", "precision"): ("f32", "f64"),
    ("bc", "dirichlet_value"): ("zero", "constant"),
    ("physics", "force"): ("none", "constant"),
    ("physics", "closure"): ("none", "smagorinsky", "vreman", "qr", "wale", "sigma", "s3pqr"),
    ("solver", "kind"): ("spectral", "direct", "cg", "fft-tridiag"),
    ("time", "method"): ("ssp33", "wray3", "rk4"),
    ("study", "profile"): ("uniform", "tanh"),
}
for _ax in "xyz":
    CHOICES[("grid", f"{_ax}_kind")] = _PROFILES
    CHOICES[("bc", _ax)] = _BCS


class RunConfig:
    """The validated, default-filled configuration ((section, key) -> value)."""

    def __init__(self, values):
        self.values = values

    def __getitem__(self, key):
        return self.values[key]

    def get(self, section, key):
        return self.values[(section, key)]

    def __eq__(self, other):
        return isinstance(other, RunConfig) and self.values == other.values


def _line_numbers(text):
    """1-based line of every section header and key (error messages)."""
    where, section = {}, None
    for no, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line[0] in "#;":
            continue
        if line[0] == "[" and line[-1] == "]":
            section = line[1:-1].strip()
            where[("__section__", section)] = no
        elif section is not None and "=" in line:
            where[(section, line.split("=", 1)[0].strip())] = no
    return where


def parse_config(text, overrides=()):
    """INI text plus ``section.key=value`` overrides -> RunConfig."""
    ini = configparser.ConfigParser(interpolation=None)
    try:
        ini.read_string(text)
    except configparser.Error as exc:
        raise ConfigurationError(f"malformed config: {exc}")
    where = _line_numbers(text)
    given = {}
    for section in ini.sections():
        if section not in SCHEMA:
            raise ConfigurationError(f"unknown section [{section}] (line {where.get(('__section__', section), '?')})")
        for key, value in ini.items(section):
            if key not in SCHEMA[section]:
                raise ConfigurationError(f"unknown key {section}.{key} (line {where.get((section, key), '?')})")
            given[(section, key)] = (value, where.get((section, key), "?"))
    for item in overrides:
        lhs, eq, value = item.partition("=")
        if not eq or "." not in lhs:
            raise ConfigurationError(f"override must look like section.key=value: {item!r}")
        section, key = (part.strip() for part in lhs.split(".", 1))
        if key not in SCHEMA.get(section, {}):
            raise ConfigurationError(f"unknown key {section}.{key} (from --set)")
        given[(section, key)] = (value.strip(), "--set")
    values = {}
    for section, keys in SCHEMA.items():
        for key, (conv, default) in keys.items():
            if (section, key) not in given:
                if default is None:
                    raise ConfigurationError(f"missing required key {section}.{key}")
                values[(section, key)] = default
                continue
            text_value, line = given[(section, key)]
            try:
                values[(section, key)] = conv(text_value)
            except (TypeError, ValueError):
                raise ConfigurationError(f"bad value for {section}.{key} (line {line}): {text_value!r}")
    for (section, key), allowed in CHOICES.items():
        if values[(section, key)] not in allowed:
            raise ConfigurationError(f"{section}.{key} must be one of {allowed}, got {values[(section, key)]!r}")
    _check(values)
    return RunConfig(values)


def _check(v):
    dim = v[("grid", "dim")]
    if dim not in (2, 3):
        raise ConfigurationError(f"grid.dim must be 2 or 3, got {dim}")
    axes = "xyz"[:dim]
    kind = v[("solver", "kind")]
    if kind == "spectral":
        if any(v[("bc", ax)] != "periodic" for ax in axes):
            raise ConfigurationError("solver.kind=spectral requires periodic boundaries on every axis")
        if any(v[("grid", f"{ax}_kind")] != "uniform" for ax in axes):
            raise ConfigurationError("solver.kind=spectral requires uniform grids on every axis")
    if kind == "fft-tridiag" and (dim != 3 or [v[("bc", ax)] == "periodic" for ax in axes] != [True, False, True]):
        raise ConfigurationError("solver.kind=fft-tridiag requires a 3D channel (periodic x/z, walls on y)")
    for ax in axes:
        if v[("grid", f"{ax}_n")] < 1:
            raise ConfigurationError(f"grid.{ax}_n must be positive, got {v[('grid', f'{ax}_n')]}")
        if v[("grid", f"{ax}_a")] >= v[("grid", f"{ax}_b")]:
            raise ConfigurationError(f"grid.{ax}_a must be below grid.{ax}_b")
    dt = v[("time", "dt")]
    if dt != "adaptive" and dt <= 0:
        raise ConfigurationError("time.dt must be positive or 'adaptive'")
    dev = v[("run", "device")]
    if not (dev == "cuda" or (dev.startswith("cuda:") and dev[5:].isdigit())):
        raise ConfigurationError(f"run.device must be 'cuda' or 'cuda:N', got {dev!r}")


def _text(value):
    if isinstance(value, tuple):
        return ", ".join(repr(x) for x in value)
    return repr(value) if isinstance(value, float) else str(value)


def emit_config(cfg):
    """The effective configuration as INI text (re-parses to ``cfg``)."""
    out = io.StringIO()
    for section, keys in SCHEMA.items():
        out.write(f"[{section}]\n")
        for key in keys:
            out.write(f"{key} = {_text(cfg.get(section, key))}\n")
        out.write("\n")
    return out.getvalue()


def build_setup(cfg):
    """cli.py:76-110 on the device path: the grid, BCs, closure, solver and
    stepper a configuration describes, on ``run.device``."""
    import torch

    from .bcs import BoundarySpec, Dirichlet, Periodic, Symmetric
    from .grid import PROFILES, build_grid
    from .les import ClosureModel
    from .timestep import Setup

    dev = cfg.get("run", "device")
    torch.cuda.set_device(int(dev[5:]) if ":" in dev else 0)
    dim = cfg.get("grid", "dim")
    dtype = np.float32 if cfg.get("run", "precision") == "f32" else np.float64

    def axis(ax):
        kind = cfg.get("grid", f"{ax}_kind")
        a, b, n = cfg.get("grid", f"{ax}_a"), cfg.get("grid", f"{ax}_b"), cfg.get("grid", f"{ax}_n")
        extra = {"tanh": (cfg.get("grid", f"{ax}_gamma"),), "stretched": (cfg.get("grid", f"{ax}_s"),)}
        return PROFILES[kind](a, b, n, *extra.get(kind, ()))

    def sides(ax):
        kind = cfg.get("bc", ax)
        if kind == "periodic":
            return (Periodic(), Periodic())
        if kind == "symmetric":
            return (Symmetric(), Symmetric())
        val = cfg.get("bc", "constant_u") if cfg.get("bc", "dirichlet_value") == "constant" else 0.0
        return (Dirichlet(val), Dirichlet(val))

    bcs = BoundarySpec([sides(ax) for ax in "xyz"[:dim]])
    grid = build_grid([axis(ax) for ax in "xyz"[:dim]], bcs, dtype=dtype)
    force = cfg.get("physics", "force_vector")[:dim] if cfg.get("physics", "force") == "constant" else None
    closure = None
    if cfg.get("physics", "closure") != "none":
        c = cfg.get("physics", "closure_c")
        closure = ClosureModel(kind=cfg.get("physics", "closure"), c=None if c < 0 else c,
                               filter_rule=cfg.get("physics", "closure_filter"), p=cfg.get("physics", "closure_p"))
    tol, max_iter = cfg.get("solver", "tol"), cfg.get("solver", "max_iter")
    return Setup(grid, bcs, nu=cfg.get("physics", "nu"), force=force, closure=closure,
                 solver=cfg.get("solver", "kind"), method=cfg.get("time", "method"),
                 cfl_conv=cfg.get("time", "cfl_conv"), cfl_diff=cfg.get("time", "cfl_diff"),
                 dt_max=cfg.get("time", "dt_max"), solver_tol=None if tol <= 0 else tol,
                 solver_max_iter=None if max_iter <= 0 else max_iter)
