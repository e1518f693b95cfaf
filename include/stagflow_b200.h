/*
 * stagflow_b200.h -- C ABI of the B200 (sm_100a) time-step path of the
 * staggered finite-volume incompressible Navier--Stokes solver.
 *
 * The reference (``stagflow``, /root/reference/pkg/src/stagflow) has no FFI:
 * its operator / solver / stepper surface is Python duck typing.  Each entry
 * point below replaces one reference function (cited file:line); the Python
 * package ``paper_2604_18536_b200`` binds them with ctypes behind the
 * reference's own names.
 *
 * Conventions
 *  - Fields are the reference's *extended* arrays (one ghost layer per side),
 *    C order, axis 0 slowest: shape (n0+2, n1+2[, n2+2]).  Pointers are device
 *    pointers; ``T`` is double (SFB_F64) or float (SFB_F32) as fixed by the plan.
 *  - Velocity fields are passed as arrays of ``dim`` component pointers.
 *  - Every call is asynchronous on ``stream`` (a cudaStream_t passed as void*)
 *    unless it returns a host scalar, in which case it synchronizes ``stream``.
 *  - A plan is bound to one device and used from one host thread; after
 *    creation no call allocates device memory.
 *  - Return value: SFB_OK or an error code; sfb_last_error() gives the message
 *    (thread-local).  Codes map to the reference's exceptions:
 *      SFB_EINVAL   -> ValueError            (e.g. operators.py:142-143)
 *      SFB_ECONFIG  -> ConfigurationError    (errors.py:4-5)
 *      SFB_ENUMERIC -> NumericalError        (errors.py:17-18)
 *      SFB_ECONVERGE -> ConvergenceError     (errors.py:8-14; sfb_cg_info gives
 *                       the iterations and the residual history)
 *      SFB_ECUDA    -> RuntimeError (CUDA / cuFFT failure)
 */
#ifndef STAGFLOW_B200_H
#define STAGFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFB_ABI_VERSION 5

enum { SFB_OK = 0, SFB_EINVAL = 1, SFB_ECONFIG = 2, SFB_ENUMERIC = 3, SFB_ECUDA = 4, SFB_ECONVERGE = 5 };
enum { SFB_F64 = 0, SFB_F32 = 1 };
/* SFB_BC_HALO: ghost planes of this axis are supplied by the caller (the
 * neighbouring z-slab of a multi-GPU decomposition); DOFs as periodic. */
enum { SFB_BC_PERIODIC = 0, SFB_BC_DIRICHLET = 1, SFB_BC_SYMMETRIC = 2, SFB_BC_HALO = 3 };
enum { SFB_SOLVER_SPECTRAL = 0, SFB_SOLVER_CHANNEL = 1, SFB_SOLVER_CG = 2 };

/* Per-axis host tables, packed axis by axis, each of length n[a]+2, in this
 * order (values already rounded to the plan dtype, as grid.py:168-171 and
 * operators.py:47-84 compute them):
 *   dx, du, 1/dx, 1/du, w_lo, w_hi, own_hi, own_lo, tan_hi, tan_lo        */
#define SFB_NTAB 10

typedef struct sfb_grid_desc {
  int32_t dim;                 /* 2 or 3 (grid.py:128-129) */
  int32_t dtype;               /* SFB_F64 / SFB_F32 */
  int32_t n[3];                /* interior extents (grid.py:136) */
  int32_t bc_lo[3], bc_hi[3];  /* per-axis boundary kinds (bcs.py:47-83) */
  double val_lo[3][3];         /* constant Dirichlet values [axis][component] */
  double val_hi[3][3];
  const double* tables;        /* SFB_NTAB tables per axis, see above */
  double width0[3];            /* widths[0] per axis (poisson.py:181) */
} sfb_grid_desc;

typedef struct sfb_plan sfb_plan;
typedef struct sfb_solver sfb_solver;
typedef struct sfb_fft sfb_fft;

/* Fused RK stage (timestep.py:186-207 + operators.py:218-238):
 *   k      = momentum_rhs(y)                  on velocity DOFs
 *   k_out  = k                                (if k_out[0] != NULL)
 *   s_out  = s_in + k*cb                      (if s_out[0] != NULL; s_in NULL -> u0)
 *   y_next = u0   + k*ca                      (if y_next[0] != NULL)
 * Only DOF entries are written; ghosts are refreshed by the next projection. */
typedef struct sfb_stage_args {
  const void* y[3];
  const void* u0[3];
  const void* s_in[3];
  void* s_out[3];
  void* y_next[3];
  void* k_out[3];
  double cb, ca, nu;
  double force[3];
  /* Optional (NULL = off): contiguous interior pressure (n0*n1*n2) of the
   * projection of y (poisson.py:333-339 fused into the stage): the kernel
   * forms y - G p on the fly, so the gradient-subtract pass and the ghost fill
   * of y are skipped.  All-periodic 3D plans only. */
  const void* p_int;
  /* Optional per-DOF body force (sample_force of a callable,
   * operators.py:241-259): extended arrays, one per component (all or none);
   * replaces force[] and is added after diffusion (operators.py:228-235). */
  const void* force_field[3];
  /* Optional (NULL = off), stage 0 of a step whose state carries the previous
   * step's deferred projection: y == u0 unprojected, p_int its pressure; the
   * kernel takes the projected u0 from shared memory for the combines and
   * writes it here once (timestep.py:208-210 fused into the next stage 0). */
  void* u0_out[3];
  /* Optional (NULL = off): per-DOF closure term of the stage state (the
   * eddy-stress divergence, les.py:343-414, from sfb_eddy_stress_divergence),
   * added after the force (operators.py:236-237); extended arrays. */
  const void* closure_term[3];
} sfb_stage_args;

int sfb_abi_version(void);
const char* sfb_last_error(void);

/* Grid / BC plan: grid.py:115-223, bcs.py:47-83, operators.py:38-90. */
int sfb_plan_create(const sfb_grid_desc* desc, sfb_plan** out);
int sfb_plan_destroy(sfb_plan* plan);
/* New Dirichlet wall values ([axis][component], row-major 3x3 each side) for
 * a time-dependent, spatially uniform callable Dirichlet (fields.py:72-76,
 * evaluated by the caller at the fill time). */
int sfb_plan_set_walls(sfb_plan* plan, const double* val_lo, const double* val_hi);

/* Ghost fills: fields.py:96-140 (velocity), fields.py:81-93 (scalar). */
int sfb_fill_ghosts_velocity(sfb_plan* plan, void* const* u, void* stream);
int sfb_fill_ghosts_scalar(sfb_plan* plan, void* p, void* stream);

/* Forward stencils (operators.py:108-238).  Outputs are whole extended
 * arrays: DOFs written, everything else zeroed unless accumulate != 0. */
int sfb_divergence(sfb_plan* plan, const void* const* u, void* out, void* stream);
int sfb_pressure_gradient(sfb_plan* plan, const void* p, void* const* out, void* stream);
int sfb_convection(sfb_plan* plan, const void* const* u, void* const* out, int accumulate, void* stream);
int sfb_diffusion(sfb_plan* plan, const void* const* u, double nu, void* const* out, int accumulate, void* stream);
/* force: per-component constants (NULL = none); force_field: per-DOF
 * extended force arrays (NULL, or NULL entries = use the constant). */
int sfb_momentum_rhs(sfb_plan* plan, const void* const* u, double nu, const double* force,
                     const void* const* force_field, void* const* out, void* stream);

/* RK building blocks (timestep.py:166-214). */
int sfb_rk_stage(sfb_plan* plan, const sfb_stage_args* args, void* stream);
/* dst = base + sum_l k[l]*coef[l] on DOFs (acc.copy_from + _axpy chain);
 * base == NULL (or base[0] == NULL) means zero.  k: flat array of nk*3 component pointers, k[3*l + a]. */
int sfb_combine(sfb_plan* plan, void* const* dst, const void* const* base, int nk,
                const void* const* k, const double* coef, void* stream);
/* Wray3 register update (timestep.py:231-246): fnew *= g; u += fnew; if fold: fold *= z; u += fold. */
int sfb_wray_update(sfb_plan* plan, void* const* u, void* const* fnew, void* const* fold,
                    double g, double z, void* stream);

/* out = W_u * u on DOFs, zero elsewhere (kinetic_energy_pullback, adjoint.py:264-273). */
int sfb_weighted_scale(sfb_plan* plan, const void* const* u, void* const* out, void* stream);

/* Reductions (operators.py:284-301, timestep.py:140-163); synchronize stream. */
int sfb_kinetic_energy(sfb_plan* plan, const void* const* u, double* out, void* stream);
int sfb_weighted_inner(sfb_plan* plan, const void* const* u, const void* const* v, double* out, void* stream);
int sfb_cfl_conv(sfb_plan* plan, const void* const* u, double* out, void* stream);

/* Pressure solvers (poisson.py:152-229) and projection (poisson.py:321-341).
 * SPECTRAL: periodic uniform grids (poisson.py:167-200).
 * CHANNEL : periodic uniform x/z, walls on y; exact replacement of the
 *           DirectPoissonSolver (poisson.py:203-229) by FFT(x,z) x batched
 *           tridiagonal(y) with the weighted zero-mean gauge. */
int sfb_solver_create(sfb_plan* plan, int kind, sfb_solver** out);
/* CG: matrix-free conjugate gradient on -W L (poisson.py:232-308), any BCs
 * and stretching.  Defaults follow the reference (tol 1e-10 fp64 / 1e-5 fp32,
 * max_iter = min(10000, 10 ceil(N^(1/d)) + 10)); sfb_cg_configure overrides. */
int sfb_cg_configure(sfb_solver* s, double tol, int max_iter);
/* Iterations of the last solve and its residual history (|r| before the first
 * iteration, then after each); *count = history length. */
int sfb_cg_info(const sfb_solver* s, int* iterations, double* history, int cap, int* count);
int sfb_solver_destroy(sfb_solver* s);
/* 1 if the solver runs the hand-written FFT engine, 0 if it uses cuFFT. */
int sfb_solver_uses_own_fft(const sfb_solver* s);
/* rhs, out: contiguous interior arrays (n0, n1[, n2]); may alias. */
int sfb_solver_solve(sfb_solver* s, const void* rhs, void* out, void* stream);
/* Full projection of u in place; p_ext (extended, ghosts filled) optional. */
int sfb_project(sfb_solver* s, void* const* u, void* p_ext, void* stream);
/* First half of the projection (poisson.py:321-333: divergence -> solve) without
 * the gradient subtract: *p_int receives the solver-owned contiguous interior
 * pressure, valid until the solver's next use.  Feed it to the next
 * sfb_rk_stage (sfb_stage_args.p_int), which applies u - G p on the fly. */
int sfb_project_solve(sfb_solver* s, const void* const* u, const void** p_int, void* stream);
/* Second half of sfb_project after sfb_project_solve: u -= G p with the
 * pressure still in the solver buffer, velocity ghost fill, optional extended
 * pressure (the deferred last projection of run_steps, poisson.py:333-341). */
int sfb_project_finish(sfb_solver* s, void* const* u, void* p_ext, void* stream);
/* Number of kernels (ours) launched by sfb_project (mode 0: without, 1: with
 * the extended pressure), sfb_project_solve (2) or sfb_slab_r2c (3). */
int sfb_project_launches(const sfb_solver* s, int with_pressure);

/* Eddy-viscosity closures (les.py:58-417).  kind: 1 smagorinsky, 2 vreman,
 * 3 qr, 4 wale, 5 sigma, 6 s3pqr; c >= 0 the model constant, pexp the s3pqr
 * exponent.  u needs filled ghosts; nu_t is written on the interior of the
 * extended scalar nut (ghosts untouched). */
int sfb_closure_nut(sfb_plan* plan, int kind, double c, double pexp, const void* const* u, void* nut, void* stream);
/* out (+)= div(2 nu_t S) on the velocity DOFs (les.py:343-417); nut with
 * filled ghosts (sfb_fill_ghosts_scalar), u with filled ghosts. */
int sfb_eddy_stress_divergence(sfb_plan* plan, const void* const* u, const void* nut, void* const* out,
                               int accumulate, void* stream);
/* min and max over the interior of an extended scalar (synchronises). */
int sfb_scalar_minmax(sfb_plan* plan, const void* f, double* mn, double* mx, void* stream);

/* Channel statistics (stats.py:55-167): plane sums over the homogeneous
 * directions at every wall index j = 1..n_wall, into a device fp64 array out.
 * mode 0: raw component sums (dim x n_wall); mode 1: the 7 fluctuation
 * moments of stats.cu (7 x n_wall), u being the fluctuation field with ghosts
 * filled by the homogeneous conditions.  Deterministic two-pass sums. */
int sfb_plane_sums(sfb_plan* plan, int wall_axis, const void* const* u, int mode, double* out, void* stream);
/* u_a -= mean[a * n_wall + j - 1] at every position of wall index j (device mean). */
int sfb_sub_plane_mean(sfb_plan* plan, int wall_axis, void* const* u, const double* mean, void* stream);

/* Slab-decomposed spectral solve (multi-GPU, axis 0 split over nranks; the
 * plan's axis 0 is SFB_BC_HALO).  One projection, with the nh half-spectrum
 * columns split into K chunks so each chunk's exchange overlaps the next
 * chunk's transform:
 *   sfb_slab_r2c      : divergence -> R2C (axis 2) -> spec
 *   sfb_slab_axis1(k) : FFT axis 1 of chunk k -> xchg block k, laid out
 *                       (P, m, n1/P, w_k) (rank q's k1 range contiguous)
 *   caller            : all-to-all xchg block k -> trans block k (n0, n1/P, w_k)
 *   sfb_slab_axis0(k) : FFT axis 0 -> 1/(Lambda N) -> inverse FFT axis 0 on trans block k
 *   caller            : all-to-all back trans block k -> xchg block k
 *   sfb_slab_axis1(k, inverse) : inverse FFT axis 1 reading xchg block k -> spec
 *   sfb_slab_c2r      : C2R -> local pressure (m planes)
 *   caller            : the neighbours' pressure planes (p_slab)
 *   sfb_slab_correct  : u -= G p (uses p_halo), fill non-halo ghosts, p_ext
 * With one rank there is no exchange: axis 1 / axis 0 run on spec in place
 * (chunk arguments ignored).  (poisson.py:167-200, 321-341 split at the two
 * transposes.) */
int sfb_slab_solver_create(sfb_plan* plan, int n0_global, int rank, int nranks, sfb_solver** out);
/* xchg is NULL when nranks == 1 (no exchange; trans aliases spec).  p_slab:
 * the slab pressure (m + 3 planes: prev's last, the m local planes = p_local,
 * next's first = p_halo, next's second), the p_int of an on-the-fly stage. */
int sfb_slab_buffers(sfb_solver* s, void** spec, void** trans, void** xchg, void** p_slab, void** p_local,
                     void** p_halo);
/* Largest useful K (1 when the axis-1 length has no register FFT engine). */
int sfb_slab_max_chunks(const sfb_solver* s);
int sfb_slab_r2c(sfb_solver* s, void* const* u, void* stream);
int sfb_slab_axis1(sfb_solver* s, int chunk, int nchunks, int inverse, void* stream);
int sfb_slab_axis0(sfb_solver* s, int chunk, int nchunks, void* stream);
int sfb_slab_c2r(sfb_solver* s, void* stream);
int sfb_slab_correct(sfb_solver* s, void* const* u, void* p_ext, void* stream);

/* Pullback of the Smagorinsky closure term (les.py:343-414 with
 * les.py:90-100's nu_t) on a periodic 3D grid: out += (dE/du)^T vbar, through
 * the resolved gradients and through nu_t.  u, nut and vbar need filled
 * (periodic) ghosts; scratch holds 16 extended scalars.  No reference
 * counterpart: its tape leaves closures out (adjoint.py:374); SURVEY 8(f2). */
int sfb_closure_pullback(sfb_plan* plan, int kind, double c, const void* const* u, const void* nut,
                         const void* const* vbar, void* const* out, void* scratch, void* stream);

/* NCCL communicator of the slab decomposition (SURVEY 8(b) comm_create,
 * 8(e)).  No reference counterpart (the reference is single-process; the
 * paper's outlook).  Rank 0 calls sfb_comm_unique_id and
 * the caller broadcasts the 128 id bytes; every rank then calls
 * sfb_comm_create on its device.  NCCL is dlopen'ed (libnccl.so.2, the copy
 * already loaded by the process).  All operations are enqueued on `stream`
 * (no host synchronisation); with one rank they are device copies. */
typedef struct sfb_comm sfb_comm;
int sfb_comm_unique_id(void* id128);
int sfb_comm_create(const void* id128, int nranks, int rank, sfb_comm** out);
int sfb_comm_destroy(sfb_comm* c);
int sfb_comm_rank(const sfb_comm* c);
/* send `bytes` to peer_send and receive `bytes` from peer_recv (one group;
 * a null buffer skips that side) */
int sfb_comm_sendrecv(sfb_comm* c, const void* send, int peer_send, void* recv, int peer_recv, size_t bytes,
                      void* stream);
/* axis-0 ghost planes of nf extended slab fields with m local planes:
 * plane 0 <- prev's plane m, plane m+1 <- next's plane 1 */
int sfb_comm_halo(sfb_comm* c, void* const* fields, int nf, size_t plane_bytes, int m, void* stream);
/* equal-split all-to-all (block q of send to rank q) */
int sfb_comm_alltoall(sfb_comm* c, const void* send, void* recv, size_t bytes_per_peer, void* stream);
/* in-place device all-reduce of fp64 values: op 0 sum, 1 min, 2 max */
int sfb_comm_allreduce_f64(sfb_comm* c, double* buf, size_t count, int op, void* stream);

/* Adjoints of the ghost fills (adjoint.py:53-111): accumulate every ghost
 * entry onto its source and zero the ghosts, axes in reverse order, for the
 * plan's boundary kinds (periodic, Dirichlet, symmetric).  Any BCs. */
int sfb_fold_ghosts_velocity(sfb_plan* plan, void* const* u, void* stream);
int sfb_fold_ghosts_scalar(sfb_plan* plan, void* f, void* stream);
/* zero_non_dofs_velocity / zero_ghosts_scalar (adjoint.py:32-50). */
int sfb_zero_non_dofs_velocity(sfb_plan* plan, void* const* u, void* stream);
int sfb_zero_ghosts_scalar(sfb_plan* plan, void* f, void* stream);
/* poisson_solve_transpose (adjoint.py:236-250): out = W S W^-1 pbar on the
 * interior of extended scalars (out's ghosts zeroed); any non-slab solver. */
int sfb_solve_transpose(sfb_solver* s, const void* pbar, void* out, void* stream);
/* project_pullback (adjoint.py:335-349) of the reverse sweep of a
 * sub-diagonal tableau: r = P^T vbar is accumulated into acc (g0 += ybar_j)
 * and only the next stage cotangent kb = c1 ybar + c2 r is stored
 * (adjoint.py:400-419's combine fused); periodic grids. */
int sfb_project_pullback_kb(sfb_solver* s, void* const* vbar, void* const* acc, const void* const* ybar, double c1,
                            double c2, void* const* kb, void* stream);

/* Pullbacks (adjoint.py:114-349), periodic grids. Mutating semantics of the
 * reference are kept: divergence_pullback zeroes pbar's ghosts;
 * the velocity-cotangent pullbacks zero vbar's non-DOFs. */
int sfb_divergence_pullback(sfb_plan* plan, void* pbar, void* const* out, void* stream);
int sfb_pressure_gradient_pullback(sfb_plan* plan, void* const* vbar, void* out, void* stream);
int sfb_diffusion_pullback(sfb_plan* plan, void* const* vbar, double nu, void* const* out, void* stream);
int sfb_convection_pullback(sfb_plan* plan, void* const* vbar, const void* const* u, void* const* out, void* stream);
/* rhs_pullback (adjoint.py:253-261): out (+)= conv_pb + diff_pb, fused.
 * accumulate != 0 adds into out instead of overwriting its DOFs. */
int sfb_rhs_pullback(sfb_plan* plan, void* const* vbar, const void* const* u, double nu,
                     void* const* out, double scale, int accumulate, void* stream);
/* project_pullback (adjoint.py:335-349): out = vbar + D^T S^T G^T(-vbar). */
int sfb_project_pullback(sfb_solver* s, void* const* vbar, void* const* out, void* stream);
/* Same, with out optional (NULL) and, if acc != NULL, acc += result on DOFs
 * (the g0 accumulation of step_backward, adjoint.py:412-415, fused). */
int sfb_project_pullback_ex(sfb_solver* s, void* const* vbar, void* const* out, void* const* acc, void* stream);

/* Real FFT backend (replaces stagflow.transforms.rfftn / irfftn,
 * transforms.py:9-12, looked up by poisson.py:196,199): all axes of a
 * contiguous C-order array of shape n[0..dim-1], dim 1..3.  rfftn writes the
 * (n[0], .., n[dim-1]/2+1) half spectrum (interleaved complex); irfftn reads
 * it (left untouched) and writes the real array normalised by 1/prod(n), as
 * scipy.fft does.  2/3/5/7-smooth shapes with an even last axis run the
 * hand-written engine, others cuFFT (sfb_fft_uses_own tells which). */
int sfb_fft_create(int dim, const int* n, int dtype, sfb_fft** out);
int sfb_fft_destroy(sfb_fft* f);
int sfb_fft_uses_own(const sfb_fft* f);
int sfb_rfftn(sfb_fft* f, const void* in, void* out, void* stream);
int sfb_irfftn(sfb_fft* f, const void* in, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STAGFLOW_B200_H */
