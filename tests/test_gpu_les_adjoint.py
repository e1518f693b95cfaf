"""GPU tests of the Smagorinsky closure's pullback (csrc/les.cu
k_cpb1-3, les.closure_pullback) and of the closure-aware unrolled gradient.
The reference has no closure adjoint (its tape omits closures,
adjoint.py:374), so these follow the reference's own adjoint test protocol
instead: the FD identity <J^T vbar, du> = <vbar, (E(u + e du) - E(u - e du)) / 2e>
(checks.py:72-126), on a stretched periodic grid."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _grid(P, shape, seed=3):
    rng = np.random.default_rng(seed)
    axes = []
    for n in shape:
        w = 1.0 + 0.4 * rng.random(n)
        b = np.concatenate([[0.0], np.cumsum(w)])
        axes.append(P.AxisCoords(b * (2 * np.pi / b[-1])))
    return P.Grid(tuple(axes), (True,) * 3)


def _rand(P, g, rng):
    u = P.VelocityField(g)
    arrs = u.numpy()
    for a in range(3):
        arrs[a][1:-1, 1:-1, 1:-1] = rng.standard_normal(g.shape)
    return P.VelocityField(g, arrs)


def _dot(x, y):
    return float(sum(np.sum(a[1:-1, 1:-1, 1:-1] * b[1:-1, 1:-1, 1:-1]) for a, b in zip(x.numpy(), y.numpy())))


def _closure_term(P, cl, u):
    bcs = P.BoundarySpec.all_periodic(3)
    P.fill_ghosts_velocity(u, bcs)
    out = P.VelocityField(u.grid)
    cl.add_rhs(u, out)
    return out


def test_closure_pullback_fd_identity(P):
    g = _grid(P, (12, 10, 14))
    rng = np.random.default_rng(7)
    cl = P.ClosureModel("smagorinsky", c=0.3)
    u, du, vb = _rand(P, g, rng), _rand(P, g, rng), _rand(P, g, rng)
    gb = P.closure_pullback(cl, u.copy(), vb.copy())
    lhs = _dot(gb, du)
    eps = 1e-6
    up = P.VelocityField(g, [a + eps * b for a, b in zip(u.numpy(), du.numpy())])
    um = P.VelocityField(g, [a - eps * b for a, b in zip(u.numpy(), du.numpy())])
    ep, em = _closure_term(P, cl, up), _closure_term(P, cl, um)
    rhs = (_dot(vb, ep) - _dot(vb, em)) / (2 * eps)
    assert abs(lhs - rhs) <= 1e-7 * abs(rhs), (lhs, rhs)


def test_closure_pullback_vs_oracle(P):
    """Cell for cell against the oracle's restatement of the same pullback
    (oracle/les_np.smagorinsky_pullback, FD-pinned on CPU)."""
    from _dev import rel
    from oracle import les_np as L
    from oracle import stagflow_np as O

    g = _grid(P, (12, 10, 14))
    og = O.OGrid([ax.boundaries for ax in g.axes], (True,) * 3)
    rng = np.random.default_rng(7)
    cl = P.ClosureModel("smagorinsky", c=0.3)
    u, vb = _rand(P, g, rng), _rand(P, g, rng)
    ref = L.smagorinsky_pullback(og, u.numpy(), vb.numpy(), c=0.3)
    got = P.closure_pullback(cl, u.copy(), vb.copy()).numpy()
    sl = tuple(slice(1, n + 1) for n in g.shape)
    errs = [rel(got[a][sl], ref[a][sl]) for a in range(3)]
    assert max(errs) <= 1e-12, errs


def test_closure_pullback_accumulates_and_is_deterministic(P):
    g = _grid(P, (8, 12, 10), seed=5)
    rng = np.random.default_rng(9)
    cl = P.ClosureModel("smagorinsky")
    u, vb = _rand(P, g, rng), _rand(P, g, rng)
    a = P.closure_pullback(cl, u.copy(), vb.copy()).numpy()
    b = P.closure_pullback(cl, u.copy(), vb.copy()).numpy()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    base = _rand(P, g, rng)
    acc = P.closure_pullback(cl, u.copy(), vb.copy(), out=base.copy(), accumulate=True).numpy()
    for x, y, z in zip(acc, a, base.numpy()):
        assert np.allclose(x[1:-1, 1:-1, 1:-1], (y + z)[1:-1, 1:-1, 1:-1], rtol=1e-14, atol=1e-14)


def test_closure_pullback_rejects_other_models(P):
    g = _grid(P, (8, 8, 8))
    u = P.VelocityField(g)
    with pytest.raises(P.ConfigurationError):
        P.closure_pullback(P.ClosureModel("vreman"), u, P.VelocityField(g))


def test_unrolled_gradient_with_closure_fd_identity(P):
    """RK4 with a Smagorinsky closure, two steps: the closure-aware gradient
    of the kinetic energy against a centred difference of the forward
    (rk_step with the same closure)."""
    from paper_2604_18536_b200 import cases

    g = cases.periodic_box(16)
    bcs = P.BoundarySpec.all_periodic(3)
    cl = P.ClosureModel("smagorinsky", c=0.5)
    setup = P.Setup(g, bcs, nu=2e-3, closure=cl, solver="spectral", method="rk4")
    u0 = cases.isotropic(g, setup.solver, seed=4)
    du = cases.isotropic(g, setup.solver, seed=5)
    loss = P.KineticEnergyLoss()
    dt, nsteps = 4e-3, 2
    grad = P.unrolled_gradient(loss, u0, nsteps, dt, setup, include_closure=True)
    lhs = _dot(grad, du)

    def run(sign, eps):
        st = setup.new_state(u0=P.VelocityField(g, [a + sign * eps * b for a, b in zip(u0.numpy(), du.numpy())]))
        for _ in range(nsteps):
            P.rk_step(st, dt, P.RK4, setup.solver, setup)
        return loss.value(st.u)

    eps = 1e-5
    rhs = (run(1, eps) - run(-1, eps)) / (2 * eps)
    assert abs(lhs - rhs) <= 1e-6 * abs(rhs), (lhs, rhs)
    # the default follows the reference (closure left out of the tape): a
    # different gradient, equal to the closure-free setup's
    plain = P.unrolled_gradient(loss, u0, nsteps, dt, setup).numpy()
    setup0 = P.Setup(g, bcs, nu=2e-3, solver="spectral", method="rk4")
    ref0 = P.unrolled_gradient(loss, u0, nsteps, dt, setup0).numpy()
    for x, y in zip(plain, ref0):
        assert np.array_equal(x, y)
    assert abs(_dot(P.VelocityField(g, plain), du) - lhs) > 1e-6 * abs(lhs)
