/*
 * morphreg_sm100.h -- C-ABI of the B200 (sm_100a) semi-Lagrangian geodesic
 * shooting library (libmorphreg_sm100.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `morphreg` (/root/reference/pkg/src/morphreg): every entry point below
 * replaces one reference function (cited per declaration).  The reference is
 * pure Python/numpy with no FFI of its own; the Python facade
 * `paper_2106_08817_b200` binds these symbols with ctypes and keeps the
 * reference's Python signatures.
 *
 * Conventions
 *  - All field pointers are caller-owned CUDA DEVICE pointers, C-contiguous,
 *    structure-of-arrays: a scalar batch is [B][N], a vector batch is
 *    [B][d][N] (component c = component along axis c, as fields.py:1-5),
 *    N = n[0]*n[1] (2D, [row][col]) or n[0]*n[1]*n[2] (3D).
 *  - `dtype` selects float32 (MR_F32) or float64 (MR_F64) for every field
 *    pointer of the call.
 *  - Stream-ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *    The library never allocates device memory and never synchronises,
 *    except where a function says so.
 *  - Return codes: 0 = OK; > 0 = invalid argument (the facade raises
 *    FieldError, fields.py:16-17); < 0 = CUDA error (RuntimeError).
 *    mr_last_error() returns a message for the calling thread's last failure.
 *  - Reentrant: no global mutable state besides per-thread error text and a
 *    one-time kernel attribute setup.
 */
#ifndef MORPHREG_SM100_H
#define MORPHREG_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MR_F32 = 0, MR_F64 = 1 };

enum {
  MR_OK = 0,
  MR_EINVAL = 1,      /* bad shape / radius / pointer -> FieldError       */
  MR_ECUDA = -1       /* CUDA launch or runtime error  -> RuntimeError    */
};

/* Guard bits, one int32 per (pair, step): integrator.py:113-118 checks, in
 * order, image / momentum / velocity, each non-finite before magnitude.
 * The lowest set bit is the check the reference raises first. */
enum {
  MR_GUARD_IMAGE_NONFINITE = 1 << 0,
  MR_GUARD_IMAGE_MAGNITUDE = 1 << 1,
  MR_GUARD_MOMENTUM_NONFINITE = 1 << 2,
  MR_GUARD_MOMENTUM_MAGNITUDE = 1 << 3,
  MR_GUARD_VELOCITY_NONFINITE = 1 << 4,
  MR_GUARD_VELOCITY_MAGNITUDE = 1 << 5
};

/* Shooting scheme (Scheme, integrator.py:48-51).  The Eulerian and Hybrid
 * schemes are 2D, as in the reference. */
enum {
  MR_SCHEME_SEMI_LAGRANGIAN = 0,
  MR_SCHEME_EULERIAN = 1,
  MR_SCHEME_HYBRID = 2
};

/* Grid of a batch of independent pairs (GridGeometry, fields.py:20-38). */
typedef struct {
  int32_t ndim;   /* 2 or 3 */
  int32_t batch;  /* B >= 1 */
  int32_t n[3];   /* 2D: {H, W, 1}; 3D: {D, H, W}; every n >= 2 */
} mr_grid;

/* Truncated Gaussian (GaussianKernel, kernel.py:17-33).  `weights` is a HOST
 * pointer to the 2r+1 normalised float64 taps (GaussianKernel.weights);
 * 1 <= radius <= MR_MAX_RADIUS. */
typedef struct {
  int32_t radius;
  const double* weights;
} mr_kernel;

#define MR_MAX_RADIUS 32

/* ---- single-step operators (2D; mr_sl_step also 3D) ------------------------ */

/* v = -K * (z grad I) for every pair.  Replaces velocity_from_momentum /
 * velocity_arr (integrator.py:93-94, 124-130), i.e. gradient_arr
 * (fields.py:161-162) + smooth_vec_arr (kernel.py:82-85).
 * workspace: nullable device scratch of 2 scalars per pixel; when given, the
 * fp32 path runs as two kernels (product + axis-1 pass, then the axis-0 pass
 * over whole columns) instead of one; the result is the same operator.
 * guard: nullable int32[B]; OR-ed with the MR_GUARD_VELOCITY_* bits of v
 * (_guard, integrator.py:113-118; mr_shoot_forward guards I and z in the
 * transport step that produces them). */
int mr_velocity(int dtype, mr_grid g, mr_kernel k, const void* I, const void* z,
                void* v, int32_t* guard, void* workspace, void* stream);

/* One semi-Lagrangian step (integrator.py:193-205):
 *   plan  = bilinear_plan(Id - dt v)            fields.py:207-224
 *   I'    = B(I) + dt mu z                       integrator.py:101-102
 *   z'    = B(z) (1 - dt div v)                  integrator.py:109-110
 *   phi'  = B(phi)   (phi_in/phi_out nullable, [B][d][N])  integrator.py:202-205 */
int mr_sl_step(int dtype, mr_grid g, double dt, double mu, const void* I,
               const void* z, const void* v, void* I_next, void* z_next,
               const void* phi_in, void* phi_out, void* stream);

/* Adjoint of one semi-Lagrangian step w.r.t. (I, z, v) -- objective.py:118-147.
 * ib_acc, zb_acc must be zero-filled by the caller (scatter targets,
 * bilinear_adjoint_values fields.py:243-254); vbar is written ([B][d][N]). */
int mr_sl_step_adjoint(int dtype, mr_grid g, double dt, double mu,
                       const void* I, const void* z, const void* v,
                       const void* ibar_next, const void* zbar_next,
                       void* ib_acc, void* zb_acc, void* vbar, void* stream);

/* Adjoint of v = -K*(z grad I) -- objective.py:157-161:
 *   mbar = -K^T vbar (smooth_adjoint_vec_arr, kernel.py:48-68, 88-92)
 *   zb  += sum_c mbar_c d_c I ;  ib += G^T(mbar z) (fields.py:148-166)
 * ib/zb are read-modify-write ([B][N]).  workspace: nullable, 2 scalars per
 * pixel; when given, the fp32 path runs the axis-0 transposed FIR over whole
 * columns first (split kernels), as mr_shoot_adjoint does. */
int mr_velocity_adjoint(int dtype, mr_grid g, mr_kernel k, const void* I,
                        const void* z, const void* vbar, void* ib, void* zb,
                        void* workspace, void* stream);

/* One transport step of any Scheme with an explicit dt -- the field-level
 * single-step operations advect_image_sl / continuity_sl (scheme SL,
 * integrator.py:141-159) and advect_image_euler / continuity_euler (EULERIAN,
 * integrator.py:133-138, 154-155).  I' and z' are both written; callers of a
 * one-output reference function discard the other.  Eulerian / Hybrid are 2D. */
int mr_scheme_step(int dtype, mr_grid g, int32_t scheme, double dt, double mu,
                   const void* I, const void* z, const void* v, void* I_next,
                   void* z_next, const void* phi_in, void* phi_out, void* stream);

/* ---- array-level operators (fields.py:144-262, kernel.py:36-68) ----------- *
 * Not on the shooting hot path (the whole-loop kernels fuse them); exported so
 * the facade is a drop-in for code that calls the operators one by one.
 * 2D or 3D grids; scalar batch [B][N], vector batch [B][d][N]. */

/* axis_diff (np.gradient, fields.py:144-145) along `axis`, or its exact
 * transpose axis_diff_adjoint (fields.py:148-158) when adjoint != 0.
 * mr_axis_diff, mr_conv1d and mr_reduce also take ndim = 1 (lines; n = {N,1,1}),
 * as the reference's array operators accept any ndarray. */
int mr_axis_diff(int dtype, mr_grid g, int32_t axis, const void* a, void* out,
                 int32_t adjoint, void* stream);

/* gradient_arr (fields.py:161-162): f [B][N] -> out [B][d][N]; with
 * adjoint != 0 its transpose gradient_adjoint_arr (fields.py:165-166):
 * f = gbar [B][d][N] -> out [B][N]. */
int mr_gradient(int dtype, mr_grid g, const void* f, void* out, int32_t adjoint,
                void* stream);

/* divergence_arr (fields.py:169-170): v [B][d][N] -> out [B][N]. */
int mr_divergence(int dtype, mr_grid g, const void* v, void* out, void* stream);

/* conv1d_replicate (kernel.py:36-45) along `axis`, or its exact transpose
 * conv1d_replicate_adjoint (kernel.py:48-68) when adjoint != 0. */
int mr_conv1d(int dtype, mr_grid g, mr_kernel k, int32_t axis, const void* a,
              void* out, int32_t adjoint, void* stream);

/* bilinear_plan + bilinear_apply (fields.py:207-240; trilinear in 3D) of
 * ncomp components a [B][ncomp][N] at absolute sample coordinates
 * coords [B][d][N] (channel c = coordinate along axis c) -> out [B][ncomp][N].
 * bad: nullable int32 device flag, set to 1 when a coordinate is non-finite
 * (bilinear_plan raises FieldError, fields.py:208-209). */
int mr_interpolate(int dtype, mr_grid g, const void* coords, const void* a,
                   void* out, int32_t ncomp, int32_t* bad, void* stream);

/* bilinear_adjoint_values (fields.py:243-254): out [B][N] = B^T gbar
 * (zero-filled by the library, then scattered). */
int mr_interpolate_adjoint(int dtype, mr_grid g, const void* coords,
                           const void* gbar, void* out, int32_t* bad,
                           void* stream);

/* bilinear_coord_grad (fields.py:257-262): out [B][d][N], derivative of the
 * interpolated value w.r.t. each coordinate times the strict inside mask. */
int mr_interpolate_coord_grad(int dtype, mr_grid g, const void* coords,
                              const void* a, void* out, int32_t* bad,
                              void* stream);

/* Per-pair reductions, fp64 accumulation, deterministic order: op 0 = dot
 * (fields.py:285-288) sum a*b; op 1 = ssd (fields.py:291-295) 0.5 sum (a-b)^2;
 * op 2 = sum a^2 (b unused).  out: double[B] device. */
int mr_reduce(int dtype, mr_grid g, int32_t op, const void* a, const void* b,
              double* out, void* stream);

/* ---- whole-loop entry points (one call per shoot / gradient) -------------- */

/* Bytes of device workspace mr_shoot_forward uses: 3 scalars per voxel in 3D,
 * where the separable smoothing round-trips through it (required); 2 scalars
 * per pixel in 2D, where it holds the transposed intermediate hT of the fp32 velocity
 * (k_vel_a / k_vel_b; optional: NULL keeps the single-kernel velocity). */
size_t mr_forward_workspace_bytes(int dtype, mr_grid g);

/* shoot() for Scheme.SEMI_LAGRANGIAN (integrator.py:163-219), every pair of
 * the batch, 2D or 3D (trilinear, 3-axis smoothing).  Trajectory buffers
 * hold all n_steps+1 states:
 *   traj_I, traj_z: [T+1][B][N]; traj_v: [T+1][B][d][N];
 *   phi: nullable [B][d][N] final pull-back grid (SampleGrid);
 *   guard: nullable int32[B][T+1] (zero-filled by the library, then OR-ed).
 * traj_I[0], traj_z[0] must already hold I0, z0. dt = 1/n_steps. */
int mr_shoot_forward(int dtype, mr_grid g, mr_kernel k, double mu,
                     int32_t n_steps, void* traj_I, void* traj_z,
                     void* traj_v, void* phi, int32_t* guard, void* workspace,
                     void* stream);

/* shoot() for any Scheme (integrator.py:163-219, branches :194-201): as
 * mr_shoot_forward (which is scheme = MR_SCHEME_SEMI_LAGRANGIAN).
 * EULERIAN: I' = I + dt(-(grad I . v) + mu z), z' = z - dt div(z v);
 * HYBRID:   I' = B(I) + dt mu z,               z' = z - dt div(z v);
 * both warp phi with the bilinear plan. */
int mr_shoot_forward_scheme(int dtype, mr_grid g, mr_kernel k, int32_t scheme,
                            double mu, int32_t n_steps, void* traj_I,
                            void* traj_z, void* traj_v, void* phi,
                            int32_t* guard, void* workspace, void* stream);

/* Bytes of device workspace mr_shoot_adjoint needs for grid g (includes the
 * fixed-point accumulators of MR_OPT_DETERMINISTIC and the cost partials). */
size_t mr_adjoint_workspace_bytes(int dtype, mr_grid g);

/* Option bits of mr_shoot_adjoint_ex.  MR_OPT_DETERMINISTIC: the transport
 * adjoint scatters accumulate in 64-bit fixed point (order-independent integer
 * adds, scaled per pair by the step's max |ibar|, |zbar|), so repeated calls on
 * the same inputs give bitwise-identical gradients -- the reference's replay
 * promise (optimizer.py:5-7).  Without it the scatters are fp32 /
 * fp64 atomics (faster; last-bit run-to-run variation). */
enum { MR_OPT_DETERMINISTIC = 1 };

/* grad() reverse sweep (objective.py:91-174) given a forward trajectory:
 *   zbar0: [B][N] output dH/dz0;  J: [B][N] targets;
 *   terms: double[B][4] device output {total, data_term, v_norm, z_norm}
 *          (CostReport, objective.py:56-61, 71-88);
 *   flags: int32[B] device, set to 1 when zbar0 holds a non-finite entry
 *          (objective.py:171-173); zero-filled by the library first. */
int mr_shoot_adjoint(int dtype, mr_grid g, mr_kernel k, double mu,
                     int32_t n_steps, double lam, double rho,
                     const void* traj_I, const void* traj_z,
                     const void* traj_v, const void* J, void* zbar0,
                     double* terms, int32_t* flags, void* workspace,
                     void* stream);

/* grad() for any Scheme (objective.py:91-174, branches :124-155) over a
 * trajectory from mr_shoot_forward_scheme with the same scheme; arguments as
 * mr_shoot_adjoint (which is scheme = MR_SCHEME_SEMI_LAGRANGIAN). */
int mr_shoot_adjoint_scheme(int dtype, mr_grid g, mr_kernel k, int32_t scheme,
                            double mu, int32_t n_steps, double lam, double rho,
                            const void* traj_I, const void* traj_z,
                            const void* traj_v, const void* J, void* zbar0,
                            double* terms, int32_t* flags, void* workspace,
                            void* stream);

/* As mr_shoot_adjoint_scheme, plus `options` (MR_OPT_* bits).
 * flags[b] bit 1 (value 2): a deterministic-mode contribution was outside the
 * fixed-point range or non-finite (the facade raises). */
int mr_shoot_adjoint_ex(int dtype, mr_grid g, mr_kernel k, int32_t scheme,
                        double mu, int32_t n_steps, double lam, double rho,
                        const void* traj_I, const void* traj_z,
                        const void* traj_v, const void* J, void* zbar0,
                        double* terms, int32_t* flags, void* workspace,
                        int32_t options, void* stream);

/* Bytes of the optional mr_cost_terms workspace (per-block partials). */
size_t mr_cost_workspace_bytes(int dtype, mr_grid g);

/* cost() terms (objective.py:71-88) from a trajectory's final image and the
 * initial state: terms double[B][4] = {total, data, v_norm, z_norm}.
 * v_norm is computed as -<m0, v0> (K m0 == -v0, kernel.py:103-108).
 * ibar_seed: nullable [B][N], receives I_T - J (objective.py:107).
 * workspace: nullable (mr_cost_workspace_bytes); the fp64 sums are reduced
 * in a fixed order either way (deterministic), the workspace spreads them over
 * many blocks per pair. */
int mr_cost_terms(int dtype, mr_grid g, double lam, double rho,
                  const void* I0, const void* z0, const void* v0,
                  const void* IT, const void* J, double* terms,
                  void* ibar_seed, void* workspace, void* stream);

/* Separable replicate-border Gaussian smoothing of a scalar batch
 * (smooth_arr, kernel.py:71-73) and its exact transpose
 * (smooth_adjoint_arr, kernel.py:76-79). */
int mr_smooth(int dtype, mr_grid g, mr_kernel k, const void* a, void* out,
              int32_t adjoint, void* stream);

const char* mr_last_error(void);
const char* mr_strerror(int code);
int mr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MORPHREG_SM100_H */
