"""The run configuration (config.py:1-261 of the reference) with the B200
keys: strict keys with line numbers, defaults, enums,
cross-field rules, --set overrides, and emit -> parse round trips.  Host
logic only (no GPU)."""

import math
import re

import pytest

from paper_2604_18536_b200.config import SCHEMA, emit_config, parse_config
from paper_2604_18536_b200.errors import ConfigurationError

CHANNEL = """
[run]
study = channel-smoke
device = cuda:0
[grid]
dim = 3
y_kind = tanh
y_a = 0
y_b = 2
[bc]
y = dirichlet
[solver]
kind = fft-tridiag
[time]
method = rk4
dt = 0.002
"""


def test_defaults_and_b200_keys():
    cfg = parse_config(CHANNEL)
    assert cfg.get("run", "device") == "cuda:0"
    assert cfg.get("solver", "kind") == "fft-tridiag"
    assert cfg.get("time", "method") == "rk4"
    assert cfg.get("time", "dt") == 0.002
    assert cfg.get("grid", "x_b") == 2.0 * math.pi
    assert cfg.get("study", "channel_n") == (32, 48, 16)
    assert parse_config("[run]\nstudy = simulate\n").get("run", "device") == "cuda"


def test_emit_round_trip_and_overrides():
    cfg = parse_config(CHANNEL, overrides=["physics.nu=0.0055", "grid.x_n = 64", "time.dt=adaptive"])
    assert cfg.get("physics", "nu") == 0.0055 and cfg.get("grid", "x_n") == 64
    assert cfg.get("time", "dt") == "adaptive"
    text = emit_config(cfg)
    assert parse_config(text) == cfg
    assert emit_config(parse_config(text)) == text
    # every schema key is emitted, section by section
    assert all(f"{k} = " in text for keys in SCHEMA.values() for k in keys)


@pytest.mark.parametrize("text,fragment", [
    ("[run]\nstudy = simulate\nspeed = 3\n", "unknown key run.speed (line 3)"),
    ("[run]\nstudy = simulate\n[gpu]\nx = 1\n", "unknown section [gpu] (line 3)"),
    ("[grid]\ndim = 3\n", "missing required key run.study"),
    ("[run]\nstudy = simulate\n[grid]\nx_n = many\n", "bad value for grid.x_n (line 4)"),
    ("[run]\nstudy = fly\n", "run.study must be one of"),
    ("[run]\nstudy = simulate\n[solver]\nkind = spectral\n[bc]\nx = dirichlet\n", "requires periodic"),
    ("[run]\nstudy = simulate\n[solver]\nkind = fft-tridiag\n", "requires a 3D channel"),
    ("[run]\nstudy = simulate\ndevice = gpu0\n", "run.device must be"),
    ("[run]\nstudy = simulate\n[time]\ndt = -1\n", "time.dt must be positive"),
    ("[run]\nstudy = simulate\n[grid]\nx_a = 3\nx_b = 1\n", "grid.x_a must be below"),
])
def test_errors_name_the_key_and_line(text, fragment):
    with pytest.raises(ConfigurationError, match=re.escape(fragment)):
        parse_config(text)


def test_bad_override():
    with pytest.raises(ConfigurationError, match="section.key=value"):
        parse_config("[run]\nstudy = simulate\n", overrides=["nu=1"])
    with pytest.raises(ConfigurationError, match="from --set"):
        parse_config("[run]\nstudy = simulate\n", overrides=["run.colour=red"])
