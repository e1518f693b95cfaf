"""CPU pin of the oracle's Smagorinsky closure pullback
(oracle/les_np.smagorinsky_pullback): the FD identity of the reference's
adjoint checks (checks.py:72-126) against the oracle's own forward
(les_np.nu_t + eddy_stress_divergence, pinned to the reference's golden
vectors).  The reference has no closure adjoint (adjoint.py:374)."""

import numpy as np

from oracle import les_np as L
from oracle import stagflow_np as O


def _grid(shape, seed):
    rng = np.random.default_rng(seed)
    bounds = []
    for n in shape:
        w = 1.0 + 0.4 * rng.random(n)
        b = np.concatenate([[0.0], np.cumsum(w)])
        bounds.append(b * (2 * np.pi / b[-1]))
    return O.OGrid(bounds, (True,) * 3)


def test_smagorinsky_pullback_fd_identity():
    g = _grid((6, 5, 7), 3)
    rng = np.random.default_rng(11)
    bcs = O.periodic_bcs(3)

    def rand():
        u = g.zeros_vel()
        for a in range(3):
            u[a][g.udof(a)] = rng.standard_normal(g.shape)
        O.fill_velocity(g, bcs, u)
        return u

    def E(u):
        u = [x.copy() for x in u]
        O.fill_velocity(g, bcs, u)
        nut = np.zeros(g.ext_shape)
        nut[g.pdof()] = L.nu_t(g, u, "smagorinsky", c=0.3)
        return L.eddy_stress_divergence(g, u, nut)

    sl = tuple(slice(1, n + 1) for n in g.shape)

    def dot(x, y):
        return sum(float(np.sum(a[sl] * b[sl])) for a, b in zip(x, y))

    u, du, vb = rand(), rand(), rand()
    lhs = dot(L.smagorinsky_pullback(g, u, vb, c=0.3), du)
    eps = 1e-6
    rhs = (dot(vb, E([a + eps * b for a, b in zip(u, du)])) - dot(vb, E([a - eps * b for a, b in zip(u, du)]))) / (
        2 * eps)
    assert abs(lhs - rhs) <= 1e-8 * abs(rhs), (lhs, rhs)
