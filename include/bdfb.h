/*
 * bdfb.h -- C ABI of libbdfb: batched, per-cell adaptive, variable-order BDF
 * integration of N independent stiff ODE systems on an NVIDIA B200 (sm_100a).
 *
 * What it computes (the hot path of arXiv 2405.01713, "SUNDIALS Time
 * Integrators for Exascale Applications with Many Independent ODE Systems"):
 *   for every cell c = 0..N-1 advance   dy_c/dt = R(t, y_c) + F_c      (Eq. 1,
 *   P:91-96; split form "dU/dt = F + R" with F frozen over dt_CFD, P:196-201,
 *   P:242-247) from t0 to tf = t0 + dt_CFD with CVODE's fixed-leading-
 *   coefficient BDF of orders 1..5, modified Newton with the
 *   stopping test of Eq. 4 and a dense LU with partial pivoting
 *    or the CVDiag diagonal solver, errors measured in the WRMS
 *   norm of Eq. 3.  The step-by-step algorithm is SURVEY.md
 *   §8(c).2; DESIGN.md lists every reading of the paper it relies on.
 *
 * Paths: BDFB_MODE_PER_CELL (default) gives every cell its own h, q and
 * history (the north_star design); the paper's lockstep batch with one
 * batch-wide WRMS norm is BDFB_MODE_GLOBAL_NORM.
 *
 * Conventions for every entry point:
 *  - All functions return int: 0 = success, < 0 = error (see BDFB_E*), and
 *    never throw or abort across the ABI.  bdfb_last_error() describes the
 *    last failure on a handle.
 *  - Pointers documented "device" are CUDA device pointers on the handle's
 *    device; "host" pointers are ordinary host memory.  The caller owns every
 *    array it passes; the library owns only its workspace and model constants.
 *  - Arrays are fp64 unless stated.  State layout is YC (component-major,
 *    y[k*N + c], the coalescing order of P:290-300) unless BDFB_LAYOUT_CY
 *    (cell-major, y[c*n + k]) is given.
 *  - A handle is bound to one device and is not thread-safe; work is enqueued
 *    on the caller's CUDA stream (cudaStream_t passed as void*, NULL = legacy
 *    default stream).
 */
#ifndef BDFB_H
#define BDFB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDFB_VERSION_MAJOR 0
#define BDFB_VERSION_MINOR 1

/* ---- error codes (< 0) -------------------------------------------------- */
#define BDFB_OK 0
#define BDFB_EINVAL (-1)      /* invalid argument                           */
#define BDFB_ENOMEM (-2)      /* device allocation failed (create only)     */
#define BDFB_ECUDA (-3)       /* CUDA runtime / launch error                */
#define BDFB_ENOMODEL (-4)    /* bdfb_set_model not called / wrong n        */
#define BDFB_ENCCL (-5)       /* NCCL error (global-norm mode)              */
#define BDFB_EUNSUPPORTED (-6)

/* ---- per-cell status (mirrors CVODE return flags) ------ */
#define BDFB_CELL_OK 0
#define BDFB_CELL_TOO_MUCH_WORK 1    /* > mxstep internal steps (reading R12) */
#define BDFB_CELL_ERR_FAILURE 2      /* 7 error-test failures in one step    */
#define BDFB_CELL_CONV_FAILURE 3     /* 10 Newton convergence failures       */
#define BDFB_CELL_RHS_FAIL 4         /* unrecoverable RHS failure            */
#define BDFB_CELL_NONFINITE_INPUT 5  /* y0 or F not finite: not integrated  */

/* ---- models: "set RHS and Jacobian kernels" ----------------------------- */
#define BDFB_MODEL_LINEAR 0        /* n=1: y' = lambda y + F; params: double lambda          */
#define BDFB_MODEL_ROBERTSON 1     /* n=3: Robertson kinetics; params: double k[3]    */
#define BDFB_MODEL_NYX_KWH 2       /* n=1: Nyx-style heating/cooling, CVDiag;
                                      params: bdfb_kwh_params; aux[c] = rho [g/cm^3]          */
#define BDFB_MODEL_MECH_H2 3       /* n=10: H2/air mechanism (mechanisms/h2_lidryer.json),
                                      constant-volume reactor; aux[c] = rho; params: NULL     */
#define BDFB_MODEL_MECH_DRM19 4    /* n=22: DRM19-class CH4/air (mechanisms/drm19_class.json) */
#define BDFB_MODEL_MECH_GRI53 5    /* n=54: GRI-3.0-class CH4/air, 53 species, 325 reactions
                                      (mechanisms/gri53_class.json; config C5): generated thread-per-cell
                                      RHS, table-driven lanes Jacobian; per cell with the SPLIT kernel
                                      (dense / CVDiag / GMRES, ERK4) or in the global-norm mode; the
                                      THREAD / GROUP kernels and the DQ Jacobian: BDFB_EUNSUPPORTED */

#define BDFB_LAYOUT_YC 0
#define BDFB_LAYOUT_CY 1

#define BDFB_MODE_PER_CELL 0
#define BDFB_MODE_GLOBAL_NORM 1

/* per-cell kernel organisation for the mechanism models (bdfb_set_kernel) */
#define BDFB_KERNEL_AUTO 0     /* = SPLIT                                               */
#define BDFB_KERNEL_THREAD 1   /* one cell per thread, straight-line generated RHS/J,
                                  per-thread-slot device workspace (csrc/bdf_tpc.cuh)    */
#define BDFB_KERNEL_GROUP 2    /* one cell per group of 16/32 lanes, state in shared
                                  memory (csrc/bdf_group.cuh; round-1 design)           */
#define BDFB_KERNEL_SPLIT 3    /* slot pool in HBM, four kernels per trip: thread-per-cell
                                  control + Newton solve (K_ctl), group Jacobian (K_jac),
                                  8-lane LU (K_lu), thread-per-cell generated RHS (K_rhs)
                                  (csrc/bdf_split.cuh); bdfb_integrate is synchronous:
                                  a host launch loop, one live-count readback per 16 trips */

typedef struct bdfb_batch bdfb_batch;

/* Nyx KWH96-form heating/cooling constants. */
typedef struct {
  double z;          /* redshift                                 */
  double X, Y;       /* hydrogen / helium mass fractions          */
  double gamma_ad;   /* adiabatic index                           */
  double gph[3];     /* photo-ionisation rates H0, He0, He+ [1/s] */
  double eph[3];     /* photo-heating rates H0, He0, He+ [erg/s]  */
} bdfb_kwh_params;

typedef struct {
  int32_t qmax;      /* maximum BDF order, 1..5 (default 5)                       */
  int32_t mode;      /* BDFB_MODE_PER_CELL (default) | BDFB_MODE_GLOBAL_NORM       */
  int64_t mxstep;    /* max internal steps per cell per integrate (default 10000)  */
  double h0;         /* initial step; 0 = CVODE cvHin estimate (default 0)         */
  double hmin;       /* minimum |h| (default 0)                                    */
  double hmax;       /* maximum |h|; 0 = unlimited (default 0)                     */
} bdfb_options;

/* Aggregate statistics of the last integrate (sums over cells). */
typedef struct {
  int64_t n_cells;
  int64_t n_failed;          /* cells with status != BDFB_CELL_OK              */
  int64_t nst, nfe, nje, nsetups, nni, netf, ncfn;   /* sums over cells       */
  int64_t nst_max;           /* max over cells of nst                          */
  int64_t nfe_max;
  int64_t nli;               /* GMRES linear (Krylov) iterations summed over cells; each made one
                                RHS call for its Jv quotient, not counted in nfe (CVODE's nfeDQ) */
} bdfb_stats;

/* Optional per-cell outputs: device arrays of length N (any may be NULL). */
typedef struct {
  int32_t *status;
  int32_t *nst, *nfe, *nje, *nsetups, *nni, *netf, *ncfn;
  int32_t *q_last;
  double *h_last;
  double *t_reached;
} bdfb_cell_stats;

/* Fill *opt with the defaults above. */
void bdfb_default_options(bdfb_options *opt);

/* Create a batch of n_cells systems of size n (1..64) on CUDA device `device`.
 * rtol > 0; atol_host: host array of n values > 0 (Eq. 3; shared by
 * all cells, reading R13).  Allocates ALL workspace once (no allocation ever
 * happens in bdfb_integrate; the lesson of P:527-535).  opt may be NULL.
 * Returns BDFB_EINVAL for bad sizes/tolerances, BDFB_ENOMEM, BDFB_ECUDA.   */
int bdfb_create(bdfb_batch **out, int64_t n_cells, int32_t n, double rtol,
                const double *atol_host, const bdfb_options *opt, int32_t device);

/* Select the RHS + Jacobian kernels ("set RHS and Jacobian kernels").
 * model_id: BDFB_MODEL_*; its n must equal the batch's n (else
 * BDFB_ENOMODEL).  params/bytes: host pointer to the model's constant
 * parameters (copied), or NULL for defaults.                               */
int bdfb_set_model(bdfb_batch *b, int32_t model_id, const void *params, size_t bytes);

/* Global-norm mode across ranks (one lockstep batch over all GPUs): create
 * the library's NCCL communicator.  nccl_unique_id: host pointer to the 128
 * bytes of an ncclUniqueId created on rank 0 and broadcast by the caller;
 * ncells_total: the batch size summed over ranks (the N of Eq. 3, R14; each
 * rank's n_cells should be a multiple of 256 so the reduction order matches
 * the single-GPU order).  Only valid for BDFB_MODE_GLOBAL_NORM handles.      */
int bdfb_set_comm(bdfb_batch *b, const void *nccl_unique_id, int32_t nranks, int32_t rank,
                  int64_t ncells_total);

/* Choose the per-cell kernel organisation (BDFB_KERNEL_*) for the mechanism
 * models; other models ignore it.  May be called before or after
 * bdfb_set_model; the THREAD kernel's workspace (about 8 (12 n + 2 n^2)
 * bytes per resident thread: Nordsieck history, weights, J, LU) is
 * allocated here or in bdfb_set_model, never in bdfb_integrate.
 * Both kernels run the same algorithm; they differ in the WRMS summation
 * order (reading R15, see bdfb_wrms_group) and hence in rounding.
 * Returns BDFB_EINVAL for an unknown id, BDFB_ENOMEM.                       */
int bdfb_set_kernel(bdfb_batch *b, int32_t kernel);

/* Jacobian of the Newton matrix M = I - gamma J:
 * BDFB_JAC_ANALYTIC (default; the paper's approaches 2A/2B) or
 * BDFB_JAC_DQ, CVODE's difference-quotient dense Jacobian (approaches 3A/3B,
 * P:399-401): column j from f(t, y + inc_j e_j) with inc_j = max(sqrt(u)|y_j|,
 * minInc/ewt_j), minInc = 1000 |h| u n ||f||_WRMS -- n extra RHS evaluations
 * per Jacobian (not counted in nfe, as in CVODE).  DQ is available for the
 * mechanism models with the SPLIT kernel in per-cell mode (else
 * BDFB_EUNSUPPORTED); BDFB_EINVAL for an unknown mode.  Call after
 * bdfb_set_model / bdfb_set_kernel.                                         */
#define BDFB_JAC_ANALYTIC 0
#define BDFB_JAC_DQ 1
int bdfb_set_jacobian(bdfb_batch *b, int32_t mode);

/* Linear solver of the Newton iteration (Table 1):
 *  BDFB_LS_DENSE (default): modified Newton with the dense LU with partial pivoting of M = I - gamma J
 *    (approaches 2A/2B with the analytic J, 3A/3B with BDFB_JAC_DQ).
 *  BDFB_LS_DIAG: CVDiag, the diagonal difference-quotient approximation of J from one extra RHS call per
 *    setup, M^-1 applied elementwise and updated exactly when gamma moves (the Nyx solver, here for
 *    any n).  The setup's RHS call is counted in nfe and as one nje.
 *  BDFB_LS_GMRES: inexact Newton-Krylov (approaches 1A/1B): no matrix setup, every Newton
 *    iteration solves (I - gamma J) delta = -G by GMRES on the scaled system of Eq. 5 (S1 = S2 = diag of the
 *    Eq. 3 weights, no preconditioner), stopping test Eq. 6 with c_l = 0.05 on the rotation residual,
 *    J v by the difference quotient (f(y + sigma v) - f(y)) / sigma, sigma = 1 / ||v||_WRMS, at the current
 *    Newton iterate; at most maxl Krylov iterations (1..5; 0 = 5, CVODE's default), no restarts.  Each
 *    Krylov iteration is one RHS call (bdfb_stats.nli), not counted in nfe.
 * DIAG and GMRES run in the SPLIT kernel of the mechanism models in per-cell mode (else BDFB_EUNSUPPORTED;
 * BDFB_EINVAL for an unknown id, maxl out of range or a DQ Jacobian mode).  The slot pool is re-sized here
 * (never in bdfb_integrate).  Readings R29 fix the details the paper leaves open.             */
#define BDFB_LS_DENSE 0
#define BDFB_LS_DIAG 1
#define BDFB_LS_GMRES 2
int bdfb_set_linear_solver(bdfb_batch *b, int32_t ls, int32_t maxl);

/* Time-integration method:
 *  BDFB_METHOD_BDF (default): the variable-order BDF of this header.
 *  BDFB_METHOD_ERK4: explicit adaptive Runge-Kutta, "a fourth-order explicit method" from ARKODE
 *    (P:415-426): the Zonneveld 5-stage 4(3) pair with the Eq. 3 WRMS error test on its embedded
 *    estimate, no algebraic solver (nje = nsetups = nni = 0, q_last = 4); one cell per thread of a
 *    persistent kernel (csrc/erk.cu), mxstep / h0 / hmin / hmax of bdfb_options apply.  Reading R30
 *     fixes the tableau and the controller constants the paper leaves open.
 * ERK4 runs the mechanism models in per-cell mode (else BDFB_EUNSUPPORTED); its workspace (8 n doubles per
 * resident thread) is allocated here.  Call after bdfb_set_model.                                        */
#define BDFB_METHOD_BDF 0
#define BDFB_METHOD_ERK4 1
int bdfb_set_method(bdfb_batch *b, int32_t method);

/* The lane-group size G whose WRMS summation order (reading R15: lane l sums
 * components i = l (mod G) in increasing i, then an xor butterfly G/2..1)
 * the selected model/kernel uses; 1 = plain sequential sum.  0 if no model
 * is set.  The oracle reproduces the order from this value.                */
int32_t bdfb_wrms_group(const bdfb_batch *b);

/* Attach (or detach with NULL) caller-owned per-cell statistics arrays that
 * the next bdfb_integrate fills.  The struct is copied.                     */
int bdfb_set_cell_stats(bdfb_batch *b, const bdfb_cell_stats *cs);

/* Integrate every cell from t0 to tf (tf > t0) on `stream`.
 *  y     : device, in/out, N*n fp64 (layout as given).  On return each cell
 *          holds y(tf), or, if its status is not OK, its last accepted state
 *          (t_reached < tf).
 *  f_ext : device, N*n fp64 frozen forcing F (same layout), or NULL for 0.
 *  aux   : device, N fp64 per-cell auxiliary input (density for NYX_KWH and
 *          MECH_*), or NULL when the model needs none.
 * Per-cell mode with a persistent kernel (THREAD, GROUP, the small models)
 * enqueues asynchronously; results are valid when `stream` completes.  The
 * SPLIT kernel (the default for MECH_*) drives its kernel launches from the
 * host in batches and returns when all cells are done (one 8-byte live-count
 * read back per batch).  Returns 0 on success / enqueue, < 0 on an argument
 * or launch error (BDFB_EUNSUPPORTED for a DQ Jacobian without SPLIT).
 * Failed cells are counted by bdfb_get_stats (they are not an error here).
 * Global-norm mode (group models only: MECH_H2, MECH_DRM19) runs the
 * integrator's control loop on the host and returns when done; its
 * statistics are batch counters (one step count for the whole batch) and a
 * failure fails every cell of the batch (R18).                              */
int bdfb_integrate(bdfb_batch *b, double t0, double tf, double *y, const double *f_ext,
                   const double *aux, int32_t layout, void *stream);

/* End-to-end variant with HOST buffers (same layout and meaning as
 * bdfb_integrate): copies y, f_ext, aux host->device, integrates and copies
 * y device->host, all on `stream`, then synchronises it.  Host buffers should
 * be page-locked for full PCIe/C2C bandwidth.  The device staging buffers
 * are allocated on the first call and kept until bdfb_destroy.            */
int bdfb_integrate_host(bdfb_batch *b, double t0, double tf, double *y_host, const double *f_ext_host,
                        const double *aux_host, int32_t layout, void *stream);

/* Synchronise the last integrate's stream and return its aggregate
 * statistics in *agg (host).  Return value: number of failed cells (>= 0)
 * or < 0 on error.                                                          */
int64_t bdfb_get_stats(bdfb_batch *b, bdfb_stats *agg);

/* Kernel launches made by the last bdfb_integrate (for bench accounting):
 * 1 for the persistent PER_CELL kernels (THREAD, GROUP); for SPLIT and in
 * GLOBAL_NORM mode every device kernel the host loop issued (NCCL's own
 * kernels excluded). */
int32_t bdfb_last_launch_count(const bdfb_batch *b);

/* Device time per kernel phase of the last bdfb_integrate with the SPLIT
 * kernel, summed over its launches and measured with CUDA events on the
 * launch stream: ms[0] K_ctl (control + Newton solve), ms[1] K_jac,
 * ms[2] K_lu, ms[3] K_rhs.  Writes min(count, max) values to ms (host, may
 * be NULL) and returns the number of phases (0 for the other kernels).     */
int32_t bdfb_phase_ms(const bdfb_batch *b, double *ms, int32_t max);

/* Device time in milliseconds of the last integrate's main kernel, measured
 * with CUDA events on the launch stream (synchronises that stream).  In
 * GLOBAL_NORM mode: the whole host-driven kernel sequence.                 */
double bdfb_last_kernel_ms(bdfb_batch *b);

/* ---- typical-value tolerances (Eq. 7; §8(f) row f2) ----------
 * "typical values" y~_i = (min(y_i) + max(y_i)) / 2 "taken over the entire
 * computational domain", atol_i = eta y~_i (eta = 1e-10 is Pele's default,
 * P:334), floored at a positive `floor` (the paper leaves y~_i = 0
 * undefined).
 *
 * bdfb_minmax: ymin[k], ymax[k] (device, n doubles each) = min and max of
 * component k over the handle's n_cells cells of y (device, `layout`),
 * with C99 fmin/fmax semantics (NaN entries are skipped).  Exact: the
 * result is independent of the reduction order except for the sign of a
 * zero.  On several ranks, reduce ymin/ymax with MIN/MAX across ranks
 * (e.g. torch.distributed.all_reduce) before the next call.
 * bdfb_set_atol_typical: tv_k = (ymin_k + ymax_k) / 2 (written to tv,
 * device, if not NULL) and the handle's atol_k = max(eta tv_k, floor); takes
 * effect for the next integrate on the same stream.  Both enqueue on
 * `stream` and return BDFB_EINVAL / BDFB_ECUDA on bad arguments / launch
 * failure.                                                                  */
int bdfb_minmax(bdfb_batch *b, const double *y, int32_t layout, double *ymin, double *ymax, void *stream);
int bdfb_set_atol_typical(bdfb_batch *b, const double *ymin, const double *ymax, double eta, double floor_,
                          double *tv, void *stream);

/* Free everything owned by the handle (NULL is a no-op). */
void bdfb_destroy(bdfb_batch *b);

/* Message for the last failure on b (or a global message when b is NULL). */
const char *bdfb_last_error(const bdfb_batch *b);

/* "MAJOR.MINOR sm_100a" */
const char *bdfb_version(void);

/* ---- diagnostic entry points: the hot path's building blocks on identical
 * inputs, for the RHS / Jacobian / LU parity tests.
 * They run the SAME device functions the integrator uses.                  */

/* f = R(t, y) + F for every cell (YC layout).  status: device int32[N] or
 * NULL (0 = ok, 1 = recoverable RHS failure).  BDFB_EINVAL if the model
 * needs aux (NYX_KWH, MECH_*) and aux is NULL (also for bdfb_eval_jac).     */
int bdfb_eval_rhs(bdfb_batch *b, double t, const double *y, const double *f_ext,
                  const double *aux, double *f, int32_t *status, void *stream);

/* J = dR/dy for every cell: J[(i*n + j)*N + c] (device, N*n*n fp64).
 * Only for dense-solver models (not NYX_KWH).  Mechanism models with the
 * SPLIT (or AUTO) kernel and the analytic Jacobian run the SPLIT path's
 * K_jac code: the two-pass generated Jacobian (reaction parts, the ordered
 * production-rate sum, one column per thread), with its device scratch
 * allocated and freed on `stream`; a cell whose T <= 0 keeps its J entries. */
int bdfb_eval_jac(bdfb_batch *b, double t, const double *y, const double *aux, double *J,
                  void *stream);

/* Batched LU with partial pivoting + solve, the integrator's own routine
 * (listing LU_FACTOR / LU_SOLVE).  For each of N systems of size
 * n (n in 1..32; n >= 5 runs the thread-per-cell routine of the mechanism
 * integrator, n <= 4 the shared-memory routine of the small models):
 * M[(i*n + j)*N + c] (device, in/out: the LU factors in
 * LAPACK getrf form, rows in pivoted order), piv[k*N + c] (device int32,
 * getrf pivot indices), b[i*N + c] (device, in/out: the solution),
 * info[c] (device int32: 0, or k+1 when pivot k is exactly zero).           */
int bdfb_lu_factor_solve(int32_t n, int64_t N, double *M, int32_t *piv, double *b,
                         int32_t *info, void *stream);

/* The SAME batched LU factor + solve as the default SPLIT integrator's hot
 * path (listing LU_FACTOR / LU_SOLVE; reading R16): oct_factor
 * (8 lanes per cell, rows in registers, as the K_lu kernel) into K_lu's
 * column-major record, then the thread-level forward/back substitutions of
 * K_ctl's Newton solve.  Arguments and layouts as bdfb_lu_factor_solve;
 * n in {2, 4, 6, 8, 10, 12, 16, 22, 32} (else BDFB_EUNSUPPORTED).  Uses
 * stream-ordered device scratch (N records) for the duration of the call.   */
int bdfb_split_lu_factor_solve(int32_t n, int64_t N, double *M, int32_t *piv, double *b,
                               int32_t *info, void *stream);

/* FP64 roofline probe: runs a DFMA-throughput kernel (all SMs, 8 independent
 * chains per thread) for about `ms` milliseconds on `device` and returns the
 * achieved FP64 TFLOP/s (2 flops per DFMA) in *tflops and the launch's SM
 * count in *sms.  Used as the measured denominator of the FP64 roofline.   */
int bdfb_probe_fp64(int32_t device, double ms, double *tflops, int32_t *sms);

#ifdef __cplusplus
}
#endif
#endif
