/*
 * mlmcp.h — C ABI of libmlmcp.so, the B200 (sm_100a) batched implicit-Euler /
 * Parareal / MLMC-reduction library behind paper_2507_19246_b200.
 *
 * The reference (arXiv 2507.19246, /root/reference/pkg/src/mlmc_parareal) is
 * pure Python; the interfaces this ABI replaces are Python callables.  Each
 * entry point below names the reference code it stands in for:
 *
 *   mlmcp_assemble         builders models.py:217-302 and the operator
 *                          formation `model.mass + dt*model.stiffness`
 *                          timeint.py:65 (per-sample CSR values on one
 *                          shared pattern instead of dense n x n matrices)
 *   mlmcp_kl_sigma         (new input kind, config 3; no reference code)
 *   mlmcp_propagate        implicit_euler_solve timeint.py:88-111 and
 *                          propagate timeint.py:114-128 (LU factor/solve
 *                          :64-75,:110,:127 replaced by Jacobi-PCG at a
 *                          stated tolerance); batched over (sample, slice)
 *                          tasks; QoI accumulation replaces evaluate_qoi
 *                          models.py:321-344 for the FE QoI kinds
 *   mlmcp_parareal_coarse  parareal_solve coarse/update sweep
 *                          parareal.py:168-178
 *   mlmcp_parareal_defect  defect parareal.py:93-103 and the stopping test
 *                          parareal.py:198-207
 *   mlmcp_parareal_finalize states[k_used:] = fine_end[k_used:]
 *                          parareal.py:209-210
 *   mlmcp_energy           new QoI kind 1/2 a^T K a (no reference code)
 *   mlmcp_level_reduce     LevelStats accumulators SPEC.md:256-260 (absent
 *                          from the reference code)
 *
 * Conventions
 *   - Every pointer argument named *_d or documented as "device" is a device
 *     pointer owned by the caller (PyTorch tensors).  The library only keeps
 *     the sparsity pattern and scalars in the context.
 *   - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t
 *     passed as void*), except where documented (streaming-path iteration
 *     control reads a device counter back to the host).
 *   - Return 0 on success or a negative MLMCP_E* code; the message is in
 *     mlmcp_last_error() (thread-local).  Per-task solver failures are
 *     reported in status[4*slot + 0..3] = {MLMCP_ST_* code, 0-based step index
 *     (SingularSystemError.step_index timeint.py:28-30), interval, iteration
 *     (PropagatorError parareal.py:37-43)}.
 *   - A context is bound to one device and is not re-entrant across threads.
 */
#ifndef MLMCP_H
#define MLMCP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLMCP_ABI_VERSION 11

/* return codes */
#define MLMCP_OK 0
#define MLMCP_EINVAL (-22)  /* -> ValueError */
#define MLMCP_ECUDA (-5)    /* -> RuntimeError */
#define MLMCP_ENOMEM (-12)  /* -> MemoryError / workspace too small */

/* per-task status codes */
#define MLMCP_ST_OK 0
#define MLMCP_ST_NOCONV 1    /* PCG hit max_it       -> SingularSystemError */
#define MLMCP_ST_BREAKDOWN 2 /* PCG curvature <= 0    -> SingularSystemError */
#define MLMCP_ST_NONFINITE 3 /* non-finite residual   -> SingularSystemError */
#define MLMCP_ST_SINGULAR 4  /* zero pivot (direct)   -> SingularSystemError */
#define MLMCP_ST_UNSUPPORTED 5 /* task flag this path does not run -> ValueError */

/* QoI modes of a task */
#define MLMCP_QOI_NONE 0
#define MLMCP_QOI_FINAL_ENERGY 1 /* qoi[slot] = 1/2 x_T^T K x_T               */
#define MLMCP_QOI_SUM_ENERGY 2   /* qoi[slot] = sum_{g > qoi_from} W(x_g)     */
/* ELECTRICAL_ENERGY models.py:337-339 without the amplitude*dt factor (applied
 * by the caller): qoi[slot] = sum_{g > qoi_from} sin(omega t_g) x_g[qoi_index] */
#define MLMCP_QOI_ELECTRICAL 3
/* MEAN_JOULE_LOSS models.py:340-343 without the 1/(dt*T) factor:
 * qoi[slot] = sum_{g > qoi_from} (x_g - x_{g-1})^T M (x_g - x_{g-1})        */
#define MLMCP_QOI_JOULE 4

typedef struct mlmcp_ctx mlmcp_ctx;

/*
 * One propagation task: n_steps implicit-Euler steps of
 *     (M + dt K) x_{g} = M x_{g-1} + dt * sin(omega t_g) * profile,
 *     t_g = t_base + (double)g * dt,  g = k0+1 .. k0+n_steps
 * (timeint.py:78-85,108-110: the grid is anchored at an origin so that a
 * sub-interval solve is bitwise the same grid as the whole-interval solve).
 * Offsets are element offsets into the caller's state buffer `xbuf`.
 * 96 bytes, natural alignment (mirrored by a numpy structured dtype).
 */
typedef struct mlmcp_task {
  int32_t sample;   /* row of the per-sample M/K value arrays            */
  int32_t n_steps;  /* >= 0                                              */
  int64_t k0;       /* grid offset                                       */
  double dt;        /* step size                                         */
  double t_base;    /* grid origin                                       */
  int64_t x_in;     /* offset of the initial state                       */
  int64_t x_out;    /* offset of the terminal state                      */
  int64_t traj;     /* offset of (n_steps+1)*N stored states, or -1      */
  int32_t qoi_slot; /* -1: no QoI                                        */
  int32_t qoi_mode; /* MLMCP_QOI_*                                       */
  int64_t qoi_from; /* SUM_ENERGY: accumulate steps with g > qoi_from    */
  int32_t group;    /* index into `active` (Parareal sample), -1: always */
  int32_t slot;     /* index into iters / status                         */
  int32_t tag;      /* copied to status[4*slot+2..3] on failure          */
  int32_t flags;    /* MLMCP_TASK_*                                      */
  int32_t qoi_index; /* ELECTRICAL: state component of the drive current  */
  int32_t ss_slot;   /* row of xss_d (periodic steady state) for the PCG
                        initial-guess predictor, -1: none                  */
} mlmcp_task;

/* task flags */
#define MLMCP_TASK_NO_EXTRAPOLATION 1 /* PCG starts from a_n (one-step method:
                                         bitwise semigroup); default:
                                         polynomial extrapolation of the task's
                                         state history (fewer PCG iterations) */
/* Homogeneous correction solve (the fine propagator is affine, so
 * F(U^k) = F(U^{k-1}) + Phi(U^k - U^{k-1}) with Phi the propagator without
 * source; parareal.py:185-188 recomputes F(U^k) from scratch): the source term
 * is dropped, x_in holds the increment, the terminal state is ADDED to
 * xbuf[x_out .. x_out+N) (which holds the solution being corrected, F^{k-1}),
 * and the stopping rule's reference norm is max(b.B^-1.b, sum_i (M_ii
 * x_out_i)^2 / A_ii), so the correction is solved to the absolute accuracy
 * of a full solve instead of relative to its own (small) right-hand side.
 * Runs on the HBM-streaming tile kernels (structured grids; a batch that
 * carries it never takes the cluster / band / cooperative kernels); qoi_mode
 * must be MLMCP_QOI_NONE.  Other paths report MLMCP_ST_UNSUPPORTED (or
 * EINVAL for non-grid patterns). */
#define MLMCP_TASK_CORRECTION 2

/* ---- library ---------------------------------------------------------- */
int mlmcp_abi_version(void);
const char* mlmcp_last_error(void);
/* number of kernels this process launched through the library (evidence) */
uint64_t mlmcp_launch_count(void);

/* ---- context ---------------------------------------------------------- */
/* row_ptr (n_rows+1) / col (nnz) are HOST arrays (int32, CSR, columns sorted
 * per row); they are validated and copied to the device. */
int mlmcp_ctx_create(int device, int n_rows, int nnz, const int32_t* row_ptr,
                     const int32_t* col, mlmcp_ctx** out);
int mlmcp_ctx_destroy(mlmcp_ctx* ctx);
/* max_row_nnz of the pattern and the widest row count the SM-resident path
 * accepts (tasks with n_rows <= small_max_rows run one CTA per task). */
int mlmcp_ctx_info(const mlmcp_ctx* ctx, int* max_row_nnz, int* small_max_rows);
/* Assembly gather map (HOST arrays, copied): for CSR entry q the
 * contributions c in [cptr[q], cptr[q+1]) are (elem[c], mw[c], kw[c]):
 *     M_q = sum_c sigma(elem_c) * mw_c,   K_q = sum_c nu(elem_c) * kw_c. */
int mlmcp_ctx_set_assembly(mlmcp_ctx* ctx, int n_elem, int n_contrib,
                           const int32_t* cptr, const int32_t* elem,
                           const double* mw, const double* kw);
/* Region-linear operator (HOST arrays, copied; structured 2D grids only):
 * for a material layout that is constant per region, the operator
 * coefficients of interior point p are sums over the six triangles around it
 * (their regions packed 4 bits each in code[p], in increasing element order):
 *     M_c(p) = sum_e sigma_{r(e)} mw[c][e],  K_c(p) = sum_e nu_{r(e)} kw[c][e]
 * for c = C (mw[0..5]), E (mw[6..7]: triangles 2, 4), N (mw[8..9]: 3, 5),
 * NE (mw[10..11]: 4, 5), in the gather map's summation order (the same
 * doubles mlmcp_assemble writes).  With it the streaming tile kernels compute
 * A = M + dt K on the fly from the per-sample region parameters passed to
 * mlmcp_propagate / mlmcp_parareal_coarse instead of streaming the operator
 * (HBM bytes per PCG iteration 112 -> 80 per point).  n_regions = 0
 * unregisters.  Replaces the per-sample operator formation models.py:284-286
 * / timeint.py:65 for region-constant materials. */
int mlmcp_ctx_set_region_grid(mlmcp_ctx* ctx, int n_regions, const uint32_t* code,
                              const double* mw, const double* kw);
/* Per-sample region parameters from drawn parameters params_d[S][2R] =
 * (nu_0..nu_{R-1}, sigma_0..sigma_{R-1}) (models.py:69-74 keeps them
 * positive; mask_d[R] zeroes the non-conducting regions after the draw):
 * sigma_d[S][R] = sigma * mask (for mlmcp_assemble, may be NULL) and
 * rp_d[S][R][2] = (sigma * mask, nu) (for the region-linear operator, may be
 * NULL).  Stream-ordered. */
int mlmcp_region_params(int S, int R, const double* params_d, const double* mask_d,
                        double* sigma_d, double* rp_d, void* stream);
/* Force a path: 0 auto, 1 SM-resident (PCG), 2 streaming (PCG), 3 direct
 * (dense LU with partial pivoting per task, one thread per task, n_rows <=
 * MLMCP_DIRECT_MAX_ROWS; the only path for non-symmetric M + dt K, e.g. the
 * Steinmetz circuit models.py:217-249).  Auto picks direct for n_rows <=
 * MLMCP_DIRECT_MAX_ROWS, SM-resident up to small_max_rows, else streaming. */
#define MLMCP_DIRECT_MAX_ROWS 4
int mlmcp_ctx_set_path(mlmcp_ctx* ctx, int path);
/* Device time of the streaming paths' PCG-iteration launches (measurement;
 * no reference counterpart): mode 1 resets and starts accumulating (CUDA
 * events around each host-loop chunk of iteration launches), 0 stops; both
 * return the totals so far in *ms and *launches (either may be NULL). */
int mlmcp_stream_timing(mlmcp_ctx* ctx, int mode, double* ms, int64_t* launches);

/* ---- K1: assembly ------------------------------------------------------ */
/* sigma(s, e) = sigma_d[s*sigma_stride + (sigma_index_d ? sigma_index_d[e] : e)]
 * (same for nu).  Writes M_d, K_d: [S][nnz]. */
int mlmcp_assemble(mlmcp_ctx* ctx, int S, const double* sigma_d,
                   int64_t sigma_stride, const int32_t* sigma_index_d,
                   const double* nu_d, int64_t nu_stride,
                   const int32_t* nu_index_d, double* M_d, double* K_d,
                   void* stream);

/* sigma_out[s][e] = exp(log_sigma0 + scale * sum_k xi[s][k] * basis[k][e]) */
int mlmcp_kl_sigma(int S, int n_elem, int n_modes, const double* xi_d,
                   const double* basis_d, double log_sigma0, double scale,
                   double* sigma_out_d, void* stream);

/* ---- K2-K4, K6: batched implicit-Euler propagation ---------------------- */
/* Workspace bytes for mlmcp_propagate / mlmcp_parareal_coarse with n_tasks
 * tasks over S per-sample operators (0 on the SM-resident path). */
size_t mlmcp_workspace_bytes(const mlmcp_ctx* ctx, int n_tasks, int S);

/* elapsed_ns_d (optional, may be NULL): device-clock nanoseconds each task
 * held its execution slot (one CTA on the SM-resident path, one thread on the
 * direct path) are ADDED to elapsed_ns_d[slot] (propagate: task.slot; coarse
 * sweep: sample).  The executor turns these into GPU effort (SM-seconds);
 * the streaming path leaves them untouched.  QoI modes ELECTRICAL / JOULE are
 * supported on the SM-resident and direct paths (EINVAL on streaming). */

/* region_params_d (optional, may be NULL): [S][R][2] region parameters of
 * the S operators (mlmcp_region_params) when the context has a region grid:
 * the streaming tile kernels then compute the operator on the fly.
 * Streaming batches need one dt per call (EINVAL otherwise), except on the
 * band path (MLMCP_PATH_BAND), whose tasks carry their own dt: a level's fine
 * and coarse solves then go into one launch, longest tasks first. */
int mlmcp_propagate(mlmcp_ctx* ctx, int n_tasks, const mlmcp_task* tasks_d,
                    int S, const double* M_d, const double* K_d,
                    const double* region_params_d, const double* profile_d, double omega, double rtol,
                    int max_it, const double* xss_d, double* xbuf_d,
                    double* qoi_d, int32_t* iters_d, int32_t* status_d,
                    const int32_t* active_d, int64_t* elapsed_ns_d,
                    void* ws_d, size_t ws_bytes, void* stream);

/* Periodic steady state of the implicit-Euler iteration (initial-guess
 * predictor, SM-resident path): for item i with operator row sample_d[i] and
 * step dt_d[i], X_d[i] = [Re X; Im X] (2 N doubles) solves
 *     (M + dt K - e^{-i omega dt} M) X = dt * profile,
 * so that ss_g = Im(X e^{i omega t_g}) is the exact periodic solution of
 * (M + dt K) a_g = M a_{g-1} + dt sin(omega t_g) profile.  Tasks with
 * ss_slot = i then start every PCG solve from ss_{g} + the polynomial
 * extrapolation of a - ss (fewer iterations; the per-step stopping rule and
 * accuracy are unchanged).  COCG to rtol (loose, e.g. 1e-8); iters_d[i] =
 * COCG iterations (optional).  SM-resident path: one CTA per item, no
 * workspace; streaming path (meshes > 1024 rows): grid-wide COCG kernels in
 * ws_d (mlmcp_periodic_workspace_bytes), host-synchronous like
 * mlmcp_propagate.  region_params_d (optional, may be NULL): the S operators'
 * region parameters (mlmcp_region_params) when the context has a region
 * grid; the streaming kernels then apply the operator from per-class stencil
 * tables instead of streaming the CSR values of M and K (176 instead of 336
 * HBM bytes per point and COCG iteration).  EINVAL on the direct path. */
size_t mlmcp_periodic_workspace_bytes(const mlmcp_ctx* ctx, int n);
int mlmcp_periodic_state(mlmcp_ctx* ctx, int n, const int32_t* sample_d,
                         const double* dt_d, int S, const double* M_d,
                         const double* K_d, const double* region_params_d,
                         const double* profile_d,
                         double omega, double rtol, int max_it, double* X_d,
                         int32_t* iters_d, void* ws_d, size_t ws_bytes,
                         void* stream);

/* ---- K5: Parareal ------------------------------------------------------ */
/* Coarse/update sweep of iteration k (1-based) for S samples.
 *   U: [S][m+1][N] boundary states, F: [S][m+1][N] fine end states,
 *   C: [S][m][N] previous coarse values, slice_k0/slice_steps: [m] coarse
 *   grid offsets / step counts of slices 1..m (index n-1).
 * Samples with active_d[s] == 0 are skipped.  Solver failures set
 * status[4*s..] = {code, step, interval n, iteration k} and clear active[s].
 * xss_d (optional, SM-resident path): [S][2][N] periodic steady states at
 * dt_c (mlmcp_periodic_state) for the initial-guess predictor. */
int mlmcp_parareal_coarse(mlmcp_ctx* ctx, int S, int k, int m,
                          const double* M_d, const double* K_d,
                          const double* region_params_d, const double* profile_d, double omega, double dt_c,
                          double t0, const int64_t* slice_k0_d,
                          const int32_t* slice_steps_d, double rtol,
                          int max_it, double* U_d, const double* F_d,
                          double* C_d, int32_t* iters_d, int32_t* status_d,
                          const int32_t* active_d, int64_t* elapsed_ns_d,
                          const double* xss_d, void* ws_d, size_t ws_bytes,
                          void* stream);

/* Jump defect of iteration k; records defect_d[s*k_max + k-1], sets
 * k_used_d[s] = k and clears active_d[s] when defect <= tol (or k == m). */
int mlmcp_parareal_defect(mlmcp_ctx* ctx, int S, int k, int m, int k_max,
                          const double* U_d, const double* F_d, double tol,
                          int32_t* active_d, int32_t* k_used_d,
                          double* defect_d, void* stream);

/* Increments of the Parareal boundary states for correction fine solves
 * (MLMCP_TASK_CORRECTION): mode 0 snapshots D[s][n] = U[s][n] (before the
 * coarse sweep of iteration k), mode 1 forms D[s][n] = U[s][n] - D[s][n]
 * (after it), for n = k-1 .. m-1 and the active samples.  U, D: [S][m+1][N]. */
int mlmcp_parareal_delta(mlmcp_ctx* ctx, int S, int k, int m, const double* U_d, double* D_d,
                         int mode, const int32_t* active_d, void* stream);

/* Which kernels mlmcp_propagate runs a batch of n_tasks tasks over S
 * operators on (with_ss: tasks carry periodic steady states; with_rp: region
 * parameters are passed; correction: the batch carries MLMCP_TASK_CORRECTION):
 * MLMCP_PATH_*. */
#define MLMCP_PATH_DIRECT 0
#define MLMCP_PATH_SMALL 1
#define MLMCP_PATH_CLUSTER 2
#define MLMCP_PATH_BAND 3
#define MLMCP_PATH_COOP 4
#define MLMCP_PATH_TILE 5
#define MLMCP_PATH_ELL 6
int mlmcp_propagate_path(const mlmcp_ctx* ctx, int n_tasks, int S, int with_ss, int with_rp,
                         int correction);

/* U[s][n] = F[s][n] for n >= k_used[s]. */
int mlmcp_parareal_finalize(mlmcp_ctx* ctx, int S, int m, double* U_d,
                            const double* F_d, const int32_t* k_used_d,
                            void* stream);

/* ---- fused estimate launch (SM-resident path) ---------------------------- */
/* A batch of independent sequential tasks (mlmcp_propagate semantics) and/or
 * a Parareal batch (mlmcp_parareal_coarse / propagate / defect / finalize
 * semantics, parareal.py:121-220) run by ONE persistent launch with a
 * device-side scheduler: each Parareal sample's chain (coarse slice n ->
 * fine slice n+1, ..., defect, next iteration) advances as soon as its own
 * inputs are ready, its ready steps take priority over the sequential tasks,
 * and the sequential tasks fill all other SM slots.  Results are identical to
 * the separate launches.  Every task kind addresses the SAME arrays: */
typedef struct mlmcp_task_arrays {
  int n_seq;                  /* sequential tasks seq_tasks_d[0 .. n_seq)        */
  const mlmcp_task* seq_tasks_d;
  const double* xss_d;        /* periodic steady states, row = task.ss_slot     */
  double* xbuf_d;             /* states of every task (task offsets)            */
  double* qoi_d;              /* task.qoi_slot                                  */
  int32_t* iters_d;           /* task.slot: PCG iterations (summed)             */
  int32_t* status_d;          /* task.slot: 4 ints                              */
  int32_t* active_d;          /* task.group (Parareal sample), 1 on entry       */
  int64_t* elapsed_ns_d;      /* task.slot (optional)                           */
} mlmcp_task_arrays;

typedef struct mlmcp_parareal_batch {
  int S;                      /* samples (0: no Parareal)                       */
  int row0;                   /* their operators: M/K rows row0 .. row0+S-1     */
  int m;                      /* sub-intervals                                  */
  int k_max;
  double tol;
  double dt_c;
  double t0;
  const int64_t* slice_k0_d;  /* [m] coarse grid offsets                        */
  const int32_t* slice_steps_d; /* [m] coarse steps per slice                   */
  const mlmcp_task* fine_tasks_d; /* [S*m]: fine slice (s, n) at s*m + n-1,
                                     sample = row0 + s, group = s             */
  int64_t u_off;              /* U [S][m+1][N] at xbuf_d + u_off, F follows U   */
  int64_t c_tmp_off;          /* S*N scratch in xbuf_d (coarse results)         */
  double* C_d;                /* [S][m][N] previous coarse values               */
  int coarse_slot;            /* iters/status/elapsed slot of sample s's coarse
                                 solves: coarse_slot + s (status: interval n,
                                 iteration k, parareal.py:151-152)             */
  int coarse_ss;              /* steady-state row at dt_c: coarse_ss + s (-1)   */
  int32_t* k_used_d;          /* [S]                                            */
  double* defects_d;          /* [S][k_max]                                     */
} mlmcp_parareal_batch;

size_t mlmcp_fused_workspace_bytes(int S_parareal, int m, int k_max);
/* grid_ctas > 0 caps the persistent grid (e.g. a Parareal-only launch on
 * grid_ctas SM slots next to a separate sequential launch); 0: all resident
 * slots. */
int mlmcp_run_fused(mlmcp_ctx* ctx, int S, const double* M_d, const double* K_d,
                    const double* profile_d, double omega, double rtol,
                    int max_it, const mlmcp_task_arrays* arrays,
                    const mlmcp_parareal_batch* pr, int grid_ctas, void* ws_d,
                    size_t ws_bytes, void* stream);

/* ---- sample draws ------------------------------------------------------ */
/* Uniform parameters for the sample keys (seed, level, k), k = k_first ..
 * k_first + n - 1 (SPEC.md:250-254 RandomStream; models.py:305-318
 * draw_parameters):  out[i][j] = lo[j] + range[j] * U_ij, where U_i. are the
 * first P doubles of numpy.random.default_rng(SeedSequence(seed,
 * spawn_key=(level, k))) and range = hi - lo — bitwise identical to
 * rng.uniform(lo, hi).  seed, level, k < 2^64.  Device version: lo_d,
 * range_d, out_d device pointers, stream-ordered; host version: the same
 * arithmetic on the CPU (parity checks). */
int mlmcp_draw_uniform(uint64_t seed, uint64_t level, int64_t k_first, int n,
                       int P, const double* lo_d, const double* range_d,
                       double* out_d, void* stream);
int mlmcp_draw_uniform_host(uint64_t seed, uint64_t level, int64_t k_first,
                            int n, int P, const double* lo, const double* range,
                            double* out);

/* ---- K6 / K7 ----------------------------------------------------------- */
/* out[i] = 1/2 x_i^T K_{sample[i]} x_i for x_i = xbuf[x_off[i] ..]. */
int mlmcp_energy(mlmcp_ctx* ctx, int n, const int32_t* sample_d,
                 const int64_t* x_off_d, const double* xbuf_d,
                 const double* K_d, double* out_d, void* stream);

/* Y = q_l - q_lm1 over n samples (fixed order); out = {sum Y, sum Y^2,
 * mean, var} with var = (sum Y^2 - n mean^2)/(n-1). */
int mlmcp_level_reduce(int n, const double* q_l_d, const double* q_lm1_d,
                       double* out_d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MLMCP_H */
