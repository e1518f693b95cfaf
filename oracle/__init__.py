"""CPU oracle for the staggered Navier--Stokes time-step path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2604_18536_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and only as the
checker (or the timed CPU reference arm), never as the thing measured or
shipped.

``oracle.stagflow_np`` restates, in numpy, the reference package ``stagflow``
(``/root/reference/pkg/src/stagflow``) for the hot path: grid tables, ghost
fills, the forward stencils, the spectral Poisson solve, the projection, the
explicit RK steps (incl. an injected RK4 tableau) and the hand-written
pullbacks.  ``oracle.channel_np`` restates the reference's direct channel
solver as an exact FFT(x,z) x tridiagonal(y) solve.

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports
``stagflow`` from ``/root/reference`` and writes ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  The reference publishes no golden vectors
of its own; its known-answer tests (stability polynomial, spectral single
mode, channel-from-rest) are re-run against the oracle as well.
"""
