"""Hand-written pullbacks (VJP) on the GPU (mirror of adjoint.py:1-444).

Every pullback is one gather-form CUDA kernel (csrc/adjoint.cu) -- the exact
transpose of (ghost fill o forward stencil) on periodic grids, the only
boundary layout the reference's differentiable path accepts
(adjoint.py:312-316).  The reference's mutating conventions are kept:
velocity-cotangent pullbacks zero the non-DOFs of their input cotangent,
``divergence_pullback`` zeroes the ghosts of its input, and
``convection_pullback`` refills the primal's ghosts.
"""

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError
from .fields import ScalarField, VelocityField, fill_ghosts_scalar, fill_ghosts_velocity
from .operators import _plan, kinetic_energy, momentum_rhs, pressure_gradient, divergence
from .plan import get_plan, stream_ptr
from .poisson import _native_solver


def _require_periodic(bcs):
    if not all(bcs.periodic):
        raise ConfigurationError("the differentiable time-stepping path supports periodic boundaries only")


def _grid_plan(grid, bcs=None):
    from .operators import default_bcs

    return get_plan(grid, bcs if bcs is not None else default_bcs(grid)).handle


def zero_ghosts_scalar(f):
    """adjoint.py:32-37 (one plane kernel)."""
    N.call("sfb_zero_ghosts_scalar", _grid_plan(f.grid), f.data.data_ptr(), stream_ptr())
    return f


def zero_non_dofs_velocity(v):
    """adjoint.py:40-50 (one plane kernel)."""
    N.call("sfb_zero_non_dofs_velocity", _grid_plan(v.grid), N.ptr3(v.u), stream_ptr())
    return v


def fold_ghosts_scalar(f, bcs):
    """adjoint.py:53-71: adjoint of the scalar ghost fill -- every ghost is
    accumulated onto its source and zeroed, axes in reverse order (one
    kernel per axis)."""
    N.call("sfb_fold_ghosts_scalar", get_plan(f.grid, bcs).handle, f.data.data_ptr(), stream_ptr())
    return f


def fold_ghosts_velocity(v, bcs):
    """adjoint.py:74-111: adjoint of the velocity ghost fill (periodic,
    Dirichlet and symmetric sides; reversed axis order)."""
    N.call("sfb_fold_ghosts_velocity", get_plan(v.grid, bcs).handle, N.ptr3(v.u), stream_ptr())
    return v


def divergence_pullback(pbar, bcs, out=None):
    """adjoint.py:114-128"""
    _require_periodic(bcs)
    grid = pbar.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_divergence_pullback", get_plan(grid, bcs).handle, pbar.data.data_ptr(), N.ptr3(out.u), stream_ptr())
    return out


def pressure_gradient_pullback(vbar, bcs, out=None):
    """adjoint.py:131-145"""
    _require_periodic(bcs)
    grid = vbar.grid
    if out is None:
        out = ScalarField(grid)
    N.call("sfb_pressure_gradient_pullback", get_plan(grid, bcs).handle, N.ptr3(vbar.u), out.data.data_ptr(),
           stream_ptr())
    return out


def diffusion_pullback(vbar, nu, bcs, out=None):
    """adjoint.py:148-173"""
    _require_periodic(bcs)
    grid = vbar.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_diffusion_pullback", get_plan(grid, bcs).handle, N.ptr3(vbar.u), float(nu), N.ptr3(out.u),
           stream_ptr())
    return out


def convection_pullback(vbar, u, bcs, out=None):
    """adjoint.py:176-227 (gather form; refills the primal's ghosts)."""
    _require_periodic(bcs)
    grid = vbar.grid
    if out is None:
        out = VelocityField(grid)
    fill_ghosts_velocity(u, bcs)
    N.call("sfb_convection_pullback", get_plan(grid, bcs).handle, N.ptr3(vbar.u), N.ptr3(u.u), N.ptr3(out.u),
           stream_ptr())
    return out


def rhs_pullback(vbar, u, nu, bcs, out=None, accumulate=False):
    """adjoint.py:253-261: convection + diffusion pullback in one kernel."""
    _require_periodic(bcs)
    grid = vbar.grid
    if out is None:
        out = VelocityField(grid)
    fill_ghosts_velocity(u, bcs)
    N.call("sfb_rhs_pullback", get_plan(grid, bcs).handle, N.ptr3(vbar.u), N.ptr3(u.u), float(nu), N.ptr3(out.u),
           1.0, int(bool(accumulate)), stream_ptr())
    return out


def poisson_pullback(pbar, solver):
    """adjoint.py:230-233"""
    return solver.solve(pbar)


def poisson_solve_transpose(pbar, solver):
    """adjoint.py:236-250: W S W^-1 (exact on stretched grids too): the
    1/W scaling, the solve and the W scaling run natively
    (``sfb_solve_transpose``)."""
    s = _native_solver(solver, solver.bcs)
    out = ScalarField(pbar.grid, empty=True)
    N.call("sfb_solve_transpose", s.handle, pbar.data.data_ptr(), out.data.data_ptr(), stream_ptr())
    return out


def kinetic_energy_pullback(u, out=None):
    """adjoint.py:264-273"""
    grid = u.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_weighted_scale", _plan(grid), N.ptr3(u.u), N.ptr3(out.u), stream_ptr())
    return out


class KineticEnergyLoss:
    """adjoint.py:276-285"""

    def value(self, u):
        return kinetic_energy(u)

    def gradient(self, u):
        return kinetic_energy_pullback(u)


class InnerProductLoss:
    """adjoint.py:288-309 (plain inner product with a fixed field)."""

    def __init__(self, c):
        self.c = c

    def value(self, u):
        g = u.grid
        return float(sum(torch.sum(self.c.u[a][g.u_slices(a)] * u.u[a][g.u_slices(a)]).item() for a in range(g.dim)))

    def gradient(self, u):
        g = u.grid
        out = VelocityField(g)
        for a in range(g.dim):
            sl = g.u_slices(a)
            out.u[a][sl] = self.c.u[a][sl]
        return out


def project_with_tape(u, solver, bcs):
    """adjoint.py:319-332: pure projection (u is left untouched except for
    its ghost fill, as in the reference)."""
    fill_ghosts_velocity(u, bcs)
    out = u.copy()
    from .poisson import project_into

    project_into(out, solver, bcs)
    return out


def project_pullback(vbar, solver, bcs):
    """adjoint.py:335-349: vbar + D^T S^T G^T(-vbar) in one fused native call
    (gradient pullback -> weighted solve -> divergence pullback)."""
    _require_periodic(bcs)
    s = _native_solver(solver, bcs)
    out = VelocityField(vbar.grid, empty=True)
    N.call("sfb_project_pullback", s.handle, N.ptr3(vbar.u), N.ptr3(out.u), stream_ptr())
    return out


def _axpy_into(grid, dst, src, coef):
    """dst += coef*src on DOFs (one combine kernel)."""
    karr = (N.VP3 * 1)()
    karr[0] = N.ptr3(src.u)
    carr = (N.ctypes.c_double * 1)(float(coef))
    N.call("sfb_combine", _plan(grid), N.ptr3(dst.u), N.ptr3(dst.u), 1, karr, carr, stream_ptr())


class _ClosureScratch:
    closure_term = None
    nut = None


def step_forward_tape(u0, dt, tableau, solver, setup, include_closure=False):
    """adjoint.py:352-384: one projected RK step recording the stage states.
    Uses the same stage kernels as rk_step.  ``include_closure``: the stage
    RHS carries the setup's closure term like rk_step's (the reference's tape
    omits closures, adjoint.py:374)."""
    from .timestep import _closure_term, _combine, _stage
    from .poisson import project_into
    from .les import active as active_closure

    closure = setup.closure if include_closure and active_closure(setup.closure) else None
    cs = _ClosureScratch()

    bcs = setup.bcs
    grid = u0.grid
    s = tableau.stages
    fill_ghosts_velocity(u0, bcs)
    stages = []
    if tableau.subdiagonal:
        # the fused stage kernels of rk_step, each projected stage state kept
        # in its own buffer for the tape.  On periodic 3D grids (no closure)
        # the intermediate projections stop after the solve and the next stage
        # kernel forms y - G p on the fly, writing the projected y once into
        # the tape (no gradient-subtract pass); otherwise full projections
        from .timestep import _fuse_projection, _project_quiet, _project_solve

        fuse = closure is None and _fuse_projection(grid)
        acc = VelocityField(grid, empty=True)
        started = False
        cur = u0
        p_pending = None
        for j in range(s):
            yrec = VelocityField(grid, empty=True) if p_pending is not None else None
            stages.append(yrec if yrec is not None else cur)
            nxt = j + 1 < s
            yn = VelocityField(grid, empty=True) if nxt else None
            b = tableau.b[j]
            ct = _closure_term(closure, cur, cs) if closure is not None else None
            _stage(setup, cur, u0=u0, s_in=acc if started else None, s_out=acc if b != 0.0 else None,
                   y_next=yn, cb=dt * b, ca=dt * (tableau.a[j + 1][j] if nxt else 0.0), closure_term=ct,
                   p_int=p_pending, u0_out=yrec)
            started = started or b != 0.0
            p_pending = None
            if nxt:
                if fuse:
                    p_pending = _project_solve(yn, solver, bcs)
                else:
                    _project_quiet(yn, solver, bcs)
                cur = yn
        project_into(acc, solver, bcs)
        return acc, (stages, dt, tableau, closure)
    ks = []
    for j in range(s):
        if j == 0:
            yj = u0
        else:
            yj = VelocityField(grid, empty=True)
            terms = [(ks[l], dt * tableau.a[j][l]) for l in range(j) if tableau.a[j][l] != 0.0]
            _combine(grid, yj, u0, [k for k, _ in terms], [c for _, c in terms])
            project_into(yj, solver, bcs)
        stages.append(yj)
        kj = VelocityField(grid, empty=True)
        ct = _closure_term(closure, yj, cs) if closure is not None else None
        _stage(setup, yj, k_out=kj, closure_term=ct)
        ks.append(kj)
    u1 = VelocityField(grid, empty=True)
    terms = [(ks[l], dt * tableau.b[l]) for l in range(s) if tableau.b[l] != 0.0]
    _combine(grid, u1, u0, [k for k, _ in terms], [c for _, c in terms])
    project_into(u1, solver, bcs)
    return u1, (stages, dt, tableau, closure)


def _combine_into(grid, dst, terms):
    """dst = sum coef*field on DOFs (no base): one kernel."""
    from .timestep import _combine

    N.call("sfb_combine", _plan(grid), N.ptr3(dst.u), N.ptr3([None] * 3), len(terms),
           _ks(terms), (N.ctypes.c_double * max(len(terms), 1))(*[c for _, c in terms]), stream_ptr())
    _ = _combine


def _ks(terms):
    karr = (N.VP3 * max(len(terms), 1))()
    for i, (f, _) in enumerate(terms):
        karr[i] = N.ptr3(f.u)
    return karr


def _project_pullback_into(vbar, solver, bcs, out=None, acc=None):
    s = _native_solver(solver, bcs)
    N.call("sfb_project_pullback_ex", s.handle, N.ptr3(vbar.u),
           N.ctypes.byref(N.ptr3(out.u)) if out is not None else None,
           N.ctypes.byref(N.ptr3(acc.u)) if acc is not None else None, stream_ptr())


def step_backward(tape, ubar, solver, setup):
    """adjoint.py:387-422.

    For sub-diagonal tableaus (RK4) the stage cotangents are formed on the fly,
    kbar_j = dt*b_j*ybar + dt*a_{j+1,j}*ybar_{j+1} (one combine kernel, no
    zero-initialised accumulators), and ``g0 += ybar_j`` is fused into the
    projection pullback; the generic path follows the reference loop."""
    stages, dt, tableau = tape[:3]
    closure = tape[3] if len(tape) > 3 else None
    bcs = setup.bcs

    def _closure_pb(kb, j, out):
        # the closure's share of the stage RHS pullback (out += dE/du^T kb)
        if closure is not None:
            from .les import closure_pullback

            closure_pullback(closure, stages[j], kb, out=out, accumulate=True)

    grid = stages[0].grid
    s = tableau.stages
    ybar = project_pullback(ubar, solver, bcs)
    g0 = ybar.copy()
    if tableau.subdiagonal:
        kb = VelocityField(grid, empty=True)
        fb = VelocityField(grid, empty=True)
        ynext = None
        spare = None
        kb_ready = False  # kb already holds stage j's cotangent (fused into the projection pullback)
        for j in reversed(range(s)):
            if not kb_ready:
                terms = []
                if tableau.b[j] != 0.0:
                    terms.append((ybar, dt * tableau.b[j]))
                if ynext is not None and j + 1 < s and tableau.a[j + 1][j] != 0.0:
                    terms.append((ynext, dt * tableau.a[j + 1][j]))
                if not terms:
                    ynext = None
                    continue
                _combine_into(grid, kb, terms)
            kb_ready = False
            if j == 0:
                rhs_pullback(kb, stages[0], setup.nu, bcs, out=g0, accumulate=True)
                _closure_pb(kb, 0, g0)
                continue
            rhs_pullback(kb, stages[j], setup.nu, bcs, out=fb)
            _closure_pb(kb, j, fb)
            c1, c2 = dt * tableau.b[j - 1], dt * tableau.a[j][j - 1]
            if c1 != 0.0 and c2 != 0.0:
                # ybar_j = P^T fb goes into g0 and straight into the next
                # stage cotangent kb = c1 ybar + c2 ybar_j (one kernel, ybar_j
                # never stored)
                s_ = _native_solver(solver, bcs)
                N.call("sfb_project_pullback_kb", s_.handle, N.ptr3(fb.u), N.ptr3(g0.u), N.ptr3(ybar.u), float(c1),
                       float(c2), N.ptr3(kb.u), stream_ptr())
                kb_ready = True
                ynext = None
                continue
            yj = spare if spare is not None else VelocityField(grid, empty=True)
            _project_pullback_into(fb, solver, bcs, out=yj, acc=g0)
            spare = ynext
            ynext = yj
        return g0
    kbars = [None] * s
    for l in range(s):
        if tableau.b[l] != 0.0:
            kb = VelocityField(grid)
            _axpy_into(grid, kb, ybar, dt * tableau.b[l])
            kbars[l] = kb
    for j in reversed(range(s)):
        if kbars[j] is None:
            continue
        fb = rhs_pullback(kbars[j], stages[j], setup.nu, bcs)
        _closure_pb(kbars[j], j, fb)
        if j == 0:
            _axpy_into(grid, g0, fb, 1.0)
            continue
        ybar_j = project_pullback(fb, solver, bcs)
        _axpy_into(grid, g0, ybar_j, 1.0)
        for l in range(j):
            aa = tableau.a[j][l]
            if aa != 0.0:
                if kbars[l] is None:
                    kbars[l] = VelocityField(grid)
                _axpy_into(grid, kbars[l], ybar_j, dt * aa)
    return g0


def unrolled_gradient(loss, u0, n_steps, dt, setup, include_closure=False):
    """adjoint.py:425-444.  ``include_closure=True`` differentiates through
    the setup's closure too (forward stages with the closure term, its
    pullback in the reverse sweep: a-posteriori closure training); the
    default follows the reference, whose tape omits closures."""
    _require_periodic(setup.bcs)
    tableau = setup.tableau
    solver = setup.solver
    u = u0.copy()
    tapes = []
    for _ in range(n_steps):
        u, tape = step_forward_tape(u, dt, tableau, solver, setup, include_closure=include_closure)
        tapes.append(tape)
    ubar = loss.gradient(u)
    for tape in reversed(tapes):
        ubar = step_backward(tape, ubar, solver, setup)
    zero_non_dofs_velocity(ubar)
    return ubar


_ = (np, fill_ghosts_scalar, momentum_rhs, pressure_gradient, divergence)
