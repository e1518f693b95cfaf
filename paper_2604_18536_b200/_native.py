"""ctypes binding of ``libstagflow_b200.so`` (declared in include/stagflow_b200.h).

There is no fallback: if the library cannot be loaded the package import
fails, and every compute call goes through the CUDA library.
"""

import ctypes
import os

from .errors import ConfigurationError, ConvergenceError, NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
# SFB_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("SFB_LIB") or os.path.join(HERE, "libstagflow_b200.so")

SFB_OK, SFB_EINVAL, SFB_ECONFIG, SFB_ENUMERIC, SFB_ECUDA, SFB_ECONVERGE = range(6)
SFB_F64, SFB_F32 = 0, 1
SFB_BC_PERIODIC, SFB_BC_DIRICHLET, SFB_BC_SYMMETRIC, SFB_BC_HALO = 0, 1, 2, 3
SFB_SOLVER_SPECTRAL, SFB_SOLVER_CHANNEL, SFB_SOLVER_CG = 0, 1, 2
SFB_NTAB = 10
ABI_VERSION = 5

vp = ctypes.c_void_p
VP3 = vp * 3


class GridDesc(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("n", ctypes.c_int32 * 3),
        ("bc_lo", ctypes.c_int32 * 3),
        ("bc_hi", ctypes.c_int32 * 3),
        ("val_lo", (ctypes.c_double * 3) * 3),
        ("val_hi", (ctypes.c_double * 3) * 3),
        ("tables", ctypes.POINTER(ctypes.c_double)),
        ("width0", ctypes.c_double * 3),
    ]


class StageArgs(ctypes.Structure):
    _fields_ = [
        ("y", VP3),
        ("u0", VP3),
        ("s_in", VP3),
        ("s_out", VP3),
        ("y_next", VP3),
        ("k_out", VP3),
        ("cb", ctypes.c_double),
        ("ca", ctypes.c_double),
        ("nu", ctypes.c_double),
        ("force", ctypes.c_double * 3),
        ("p_int", vp),
        ("force_field", VP3),
        ("u0_out", VP3),
        ("closure_term", VP3),
    ]


# name -> argtypes (all return int status)
_SIGS = {
    "sfb_plan_create": [ctypes.POINTER(GridDesc), ctypes.POINTER(vp)],
    "sfb_plan_destroy": [vp],
    "sfb_plan_set_walls": [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    "sfb_fill_ghosts_velocity": [vp, VP3, vp],
    "sfb_fill_ghosts_scalar": [vp, vp, vp],
    "sfb_divergence": [vp, VP3, vp, vp],
    "sfb_pressure_gradient": [vp, vp, VP3, vp],
    "sfb_convection": [vp, VP3, VP3, ctypes.c_int, vp],
    "sfb_diffusion": [vp, VP3, ctypes.c_double, VP3, ctypes.c_int, vp],
    "sfb_momentum_rhs": [vp, VP3, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(VP3), VP3, vp],
    "sfb_rk_stage": [vp, ctypes.POINTER(StageArgs), vp],
    "sfb_combine": [vp, VP3, VP3, ctypes.c_int, ctypes.POINTER(VP3), ctypes.POINTER(ctypes.c_double), vp],
    "sfb_wray_update": [vp, VP3, VP3, VP3, ctypes.c_double, ctypes.c_double, vp],
    "sfb_weighted_scale": [vp, VP3, VP3, vp],
    "sfb_kinetic_energy": [vp, VP3, ctypes.POINTER(ctypes.c_double), vp],
    "sfb_weighted_inner": [vp, VP3, VP3, ctypes.POINTER(ctypes.c_double), vp],
    "sfb_cfl_conv": [vp, VP3, ctypes.POINTER(ctypes.c_double), vp],
    "sfb_solver_create": [vp, ctypes.c_int, ctypes.POINTER(vp)],
    "sfb_closure_nut": [vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, VP3, vp, vp],
    "sfb_eddy_stress_divergence": [vp, VP3, vp, VP3, ctypes.c_int, vp],
    "sfb_closure_pullback": [vp, ctypes.c_int, ctypes.c_double, VP3, vp, VP3, VP3, vp, vp],
    "sfb_scalar_minmax": [vp, vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), vp],
    "sfb_plane_sums": [vp, ctypes.c_int, VP3, ctypes.c_int, vp, vp],
    "sfb_sub_plane_mean": [vp, ctypes.c_int, VP3, vp, vp],
    "sfb_cg_configure": [vp, ctypes.c_double, ctypes.c_int],
    "sfb_cg_info": [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                    ctypes.POINTER(ctypes.c_int)],
    "sfb_solver_destroy": [vp],
    "sfb_solver_uses_own_fft": [vp],
    "sfb_solver_solve": [vp, vp, vp, vp],
    "sfb_project": [vp, VP3, vp, vp],
    "sfb_project_solve": [vp, VP3, ctypes.POINTER(vp), vp],
    "sfb_project_launches": [vp, ctypes.c_int],
    "sfb_project_finish": [vp, VP3, vp, vp],
    "sfb_slab_solver_create": [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
    "sfb_slab_buffers": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                         ctypes.POINTER(vp), ctypes.POINTER(vp)],
    "sfb_slab_r2c": [vp, VP3, vp],
    "sfb_slab_max_chunks": [vp],
    "sfb_slab_axis1": [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp],
    "sfb_slab_axis0": [vp, ctypes.c_int, ctypes.c_int, vp],
    "sfb_slab_c2r": [vp, vp],
    "sfb_slab_correct": [vp, VP3, vp, vp],
    "sfb_comm_unique_id": [vp],
    "sfb_comm_create": [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
    "sfb_comm_destroy": [vp],
    "sfb_comm_rank": [vp],
    "sfb_comm_sendrecv": [vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_size_t, vp],
    "sfb_comm_halo": [vp, VP3, ctypes.c_int, ctypes.c_size_t, ctypes.c_int, vp],
    "sfb_comm_alltoall": [vp, vp, vp, ctypes.c_size_t, vp],
    "sfb_comm_allreduce_f64": [vp, vp, ctypes.c_size_t, ctypes.c_int, vp],
    "sfb_fold_ghosts_velocity": [vp, VP3, vp],
    "sfb_fold_ghosts_scalar": [vp, vp, vp],
    "sfb_zero_non_dofs_velocity": [vp, VP3, vp],
    "sfb_zero_ghosts_scalar": [vp, vp, vp],
    "sfb_solve_transpose": [vp, vp, vp, vp],
    "sfb_divergence_pullback": [vp, vp, VP3, vp],
    "sfb_pressure_gradient_pullback": [vp, VP3, vp, vp],
    "sfb_diffusion_pullback": [vp, VP3, ctypes.c_double, VP3, vp],
    "sfb_convection_pullback": [vp, VP3, VP3, VP3, vp],
    "sfb_rhs_pullback": [vp, VP3, VP3, ctypes.c_double, VP3, ctypes.c_double, ctypes.c_int, vp],
    "sfb_project_pullback": [vp, VP3, VP3, vp],
    "sfb_project_pullback_ex": [vp, VP3, ctypes.POINTER(VP3), ctypes.POINTER(VP3), vp],
    "sfb_project_pullback_kb": [vp, VP3, VP3, VP3, ctypes.c_double, ctypes.c_double, VP3, vp],
    "sfb_fft_create": [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(vp)],
    "sfb_fft_destroy": [vp],
    "sfb_fft_uses_own": [vp],
    "sfb_rfftn": [vp, vp, vp, vp],
    "sfb_irfftn": [vp, vp, vp, vp],
}

EXPORTED = sorted(list(_SIGS) + ["sfb_abi_version", "sfb_last_error"])


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2604_18536_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    lib.sfb_abi_version.restype = ctypes.c_int
    lib.sfb_abi_version.argtypes = []
    lib.sfb_last_error.restype = ctypes.c_char_p
    lib.sfb_last_error.argtypes = []
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    if lib.sfb_abi_version() != ABI_VERSION:
        raise ImportError("libstagflow_b200.so ABI version mismatch; rebuild")
    return lib


lib = _load()


def check(rc):
    if rc == SFB_OK:
        return
    msg = lib.sfb_last_error().decode(errors="replace")
    if rc == SFB_EINVAL:
        raise ValueError(msg)
    if rc == SFB_ECONFIG:
        raise ConfigurationError(msg)
    if rc == SFB_ECONVERGE:
        raise ConvergenceError(msg)
    if rc == SFB_ENUMERIC:
        raise NumericalError(msg)
    raise RuntimeError(f"stagflow_b200 CUDA failure: {msg}")


# number of our own kernel launches each entry point issues (cuFFT's
# transforms are counted separately by the caller); used by bench.py
KERNELS_PER_CALL = {
    "sfb_rk_stage": 1, "sfb_combine": 1, "sfb_wray_update": 1, "sfb_fill_ghosts_velocity": 1,
    "sfb_fill_ghosts_scalar": 1, "sfb_divergence": 1, "sfb_pressure_gradient": 1, "sfb_convection": 1,
    "sfb_diffusion": 1, "sfb_momentum_rhs": 1, "sfb_weighted_scale": 1, "sfb_kinetic_energy": 2,
    "sfb_weighted_inner": 2, "sfb_cfl_conv": 2, "sfb_solver_solve": 1,
    "sfb_closure_nut": 1, "sfb_eddy_stress_divergence": 1, "sfb_scalar_minmax": 2,
    "sfb_plane_sums": 2, "sfb_sub_plane_mean": 1,
    "sfb_divergence_pullback": 2, "sfb_pressure_gradient_pullback": 2, "sfb_diffusion_pullback": 2,
    "sfb_convection_pullback": 2, "sfb_rhs_pullback": 2, "sfb_project_pullback": 4, "sfb_project_pullback_ex": 4,
    "sfb_fold_ghosts_velocity": 3, "sfb_fold_ghosts_scalar": 3, "sfb_zero_non_dofs_velocity": 1,
    "sfb_zero_ghosts_scalar": 1, "sfb_solve_transpose": 3,
    "sfb_slab_axis0": 1, "sfb_slab_axis1": 1, "sfb_slab_c2r": 1, "sfb_slab_correct": 2,
}
launches = 0
_FFT_PASSES = {}  # sfb_fft handle -> hand-written kernels per transform (transforms.py)


def call(name, *args):
    global launches
    check(getattr(lib, name)(*args))
    if name in ("sfb_project", "sfb_project_solve", "sfb_slab_r2c"):
        with_p = name == "sfb_project" and args[2] is not None and args[2] != 0
        mode = {"sfb_project_solve": 2, "sfb_slab_r2c": 3}.get(name, int(with_p))
        k = lib.sfb_project_launches(args[0], mode)
        launches += k
        return
    k = KERNELS_PER_CALL.get(name, 0)
    if name == "sfb_project_finish":
        k = 2 + (args[2] is not None and args[2] != 0)
    if name in ("sfb_rfftn", "sfb_irfftn"):
        # engine passes (0 on the cuFFT path) + irfftn's normalisation kernel
        k = _FFT_PASSES.get(args[0], 0) + (name == "sfb_irfftn")
    if name in ("sfb_project_pullback", "sfb_project_pullback_ex", "sfb_solver_solve", "sfb_solve_transpose"):
        own = lib.sfb_solver_uses_own_fft(args[0])
        k += 4 if own else 0
    launches += k


def ptr3(tensors):
    """VP3 of data pointers (None -> NULL)."""
    out = VP3()
    for i, t in enumerate(tensors):
        out[i] = None if t is None else t.data_ptr()
    return out
