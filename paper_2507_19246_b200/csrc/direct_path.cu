// direct_path.cu — implicit Euler for small dense systems (n <= 4): one thread
// per task, (M + dt K) factored once per task by LU with partial pivoting and
// kept in registers, then one permuted forward/back substitution per step.
//
// This is the reference's own solver (timeint.py:64-75 `_factorize`: scipy
// lu_factor; :108-110 / :126-127 `lu_solve(lu_piv, mass @ x + dt*forcing)`)
// restated for a GPU thread: pivot = first row with max |a_ik| (LAPACK
// idamax), multipliers by division, back substitution by division.  It is the
// only path for non-symmetric operators (the Steinmetz circuit,
// models.py:217-249), where PCG does not apply.  A zero pivot or a
// non-finite factor reports MLMCP_ST_SINGULAR at step 0, as timeint.py:70-74
// raises SingularSystemError(step_index=0).
//
// Register layout: the n x n factor, the dense mass matrix and the state live
// in registers (NM x NM arrays indexed only by compile-time constants; runtime
// pivots are applied by predicated selects, so nothing spills to local
// memory).
#include <cuda_runtime.h>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

struct DirectArgs {
  const mlmcp_task* tasks;
  int n_tasks;
  int n;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* M;
  const double* K;
  const double* profile;
  double omega;
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  const int32_t* active;
  int64_t* elapsed;
};

// dense [NM][NM] from the CSR values of one sample (zeros outside the pattern)
template <int NM>
__device__ __forceinline__ void load_dense(const DirectArgs& a, const double* __restrict__ v,
                                           double (&d)[NM][NM]) {
#pragma unroll
  for (int i = 0; i < NM; ++i) {
#pragma unroll
    for (int j = 0; j < NM; ++j) d[i][j] = 0.0;
    if (i < a.n) {
      const int q0 = a.row_ptr[i], q1 = a.row_ptr[i + 1];
#pragma unroll
      for (int e = 0; e < NM; ++e) {
        const int q = q0 + e;
        if (q < q1) {
          const int c = a.col[q];
          const double x = v[q];
#pragma unroll
          for (int j = 0; j < NM; ++j)
            if (c == j) d[i][j] = x;
        }
      }
    }
  }
}

// LU with partial pivoting in place; returns false on a zero pivot or a
// non-finite factor.  piv[k] = row swapped with k (LAPACK ipiv convention).
template <int NM>
__device__ __forceinline__ bool lu_factor(double (&a)[NM][NM], int (&piv)[NM], int n) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    piv[k] = k;
    if (k >= n) continue;
    int p = k;
    double best = fabs(a[k][k]);
#pragma unroll
    for (int i = k + 1; i < NM; ++i)
      if (i < n && fabs(a[i][k]) > best) {   // strict: first maximum wins
        best = fabs(a[i][k]);
        p = i;
      }
    piv[k] = p;
#pragma unroll
    for (int i = k + 1; i < NM; ++i)
      if (i == p) {
#pragma unroll
        for (int j = 0; j < NM; ++j) {
          const double t = a[k][j];
          a[k][j] = a[i][j];
          a[i][j] = t;
        }
      }
    const double pk = a[k][k];
    if (!(pk != 0.0) || !isfinite(pk)) ok = false;
#pragma unroll
    for (int i = k + 1; i < NM; ++i) {
      if (i < n) {
        const double l = a[i][k] / pk;
        a[i][k] = l;
#pragma unroll
        for (int j = k + 1; j < NM; ++j) a[i][j] = fma(-l, a[k][j], a[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NM; ++i)
#pragma unroll
    for (int j = 0; j < NM; ++j)
      if (i < n && j < n && !isfinite(a[i][j])) ok = false;
  return ok;
}

// x <- A^{-1} b with the factor of lu_factor (b permuted, L unit lower, U upper)
template <int NM>
__device__ __forceinline__ void lu_solve(const double (&a)[NM][NM], const int (&piv)[NM], int n,
                                         double (&b)[NM]) {
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    if (k >= n) continue;
#pragma unroll
    for (int i = k + 1; i < NM; ++i)
      if (i == piv[k]) {
        const double t = b[k];
        b[k] = b[i];
        b[i] = t;
      }
  }
#pragma unroll
  for (int i = 1; i < NM; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j)
      if (i < n) b[i] = fma(-a[i][j], b[j], b[i]);
#pragma unroll
  for (int i = NM - 1; i >= 0; --i) {
    if (i >= n) continue;
#pragma unroll
    for (int j = i + 1; j < NM; ++j)
      if (j < n) b[i] = fma(-a[i][j], b[j], b[i]);
    b[i] = b[i] / a[i][i];
  }
}

// 1/2 x^T V x with V the CSR values of one sample
template <int NM>
__device__ __forceinline__ double quad_form(const DirectArgs& a, const double* __restrict__ v,
                                            const double (&x)[NM]) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    if (i >= a.n) continue;
    double s = 0.0;
    for (int q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) {
      const int c = a.col[q];
      double xc = 0.0;
#pragma unroll
      for (int j = 0; j < NM; ++j)
        if (c == j) xc = x[j];
      s = fma(v[q], xc, s);
    }
    acc = fma(x[i], s, acc);
  }
  return 0.5 * acc;
}

// b = M x + dt * (sf * profile)   (timeint.py:109 operation order)
template <int NM>
__device__ __forceinline__ void rhs(const double (&m)[NM][NM], const double (&x)[NM],
                                    const double (&prof)[NM], double dt, double sf, int n,
                                    double (&b)[NM]) {
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NM; ++j)
      if (j < n) s = fma(m[i][j], x[j], s);
    b[i] = i < n ? __dadd_rn(s, __dmul_rn(dt, __dmul_rn(sf, prof[i]))) : 0.0;
  }
}

template <int NM>
__device__ __forceinline__ void factor_task(const DirectArgs& a, int sample, double dt,
                                            double (&m)[NM][NM], double (&lu)[NM][NM],
                                            int (&piv)[NM], bool& ok) {
  const double* Ms = a.M + (int64_t)sample * a.nnz;
  const double* Ks = a.K + (int64_t)sample * a.nnz;
  load_dense<NM>(a, Ms, m);
  double k[NM][NM];
  load_dense<NM>(a, Ks, k);
#pragma unroll
  for (int i = 0; i < NM; ++i)
#pragma unroll
    for (int j = 0; j < NM; ++j) lu[i][j] = op_entry(m[i][j], k[i][j], dt);
  ok = lu_factor<NM>(lu, piv, a.n);
}

template <int NM>
__global__ void __launch_bounds__(128) direct_propagate_kernel(DirectArgs a) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= a.n_tasks) return;
  const int64_t t_start = global_ns();
  const mlmcp_task t = a.tasks[tid];
  if (a.active != nullptr && t.group >= 0 && a.active[t.group] == 0) return;
  if (t.flags & MLMCP_TASK_CORRECTION) {   // tile-path-only task kind
    write_status(a.status, t.slot, MLMCP_ST_UNSUPPORTED, 0, t.tag, t.tag);
    return;
  }
  const int n = a.n;
  double m[NM][NM], lu[NM][NM], x[NM], prof[NM], b[NM], xprev[NM];
  int piv[NM];
  bool ok;
  factor_task<NM>(a, t.sample, t.dt, m, lu, piv, ok);
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    x[i] = i < n ? a.xbuf[t.x_in + i] : 0.0;
    prof[i] = i < n ? a.profile[i] : 0.0;
    if (t.traj >= 0 && i < n) a.xbuf[t.traj + i] = x[i];
  }
  const double* Ms = a.M + (int64_t)t.sample * a.nnz;
  const double* Ks = a.K + (int64_t)t.sample * a.nnz;
  double acc = 0.0;
  int code = ok ? MLMCP_ST_OK : MLMCP_ST_SINGULAR;
  if (ok) {
    for (int step = 0; step < t.n_steps; ++step) {
      const int64_t g = t.k0 + step + 1;
      const double sf = sin(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)));
      rhs<NM>(m, x, prof, t.dt, sf, n, b);
      lu_solve<NM>(lu, piv, n, b);
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        xprev[i] = x[i];
        x[i] = b[i];
      }
      if (t.traj >= 0) {
#pragma unroll
        for (int i = 0; i < NM; ++i)
          if (i < n) a.xbuf[t.traj + (int64_t)(step + 1) * n + i] = x[i];
      }
      if (g > t.qoi_from) {
        if (t.qoi_mode == MLMCP_QOI_SUM_ENERGY) {
          acc += quad_form<NM>(a, Ks, x);
        } else if (t.qoi_mode == MLMCP_QOI_JOULE) {
          double d[NM];
#pragma unroll
          for (int i = 0; i < NM; ++i) d[i] = x[i] - xprev[i];
          acc += 2.0 * quad_form<NM>(a, Ms, d);
        } else if (t.qoi_mode == MLMCP_QOI_ELECTRICAL) {
          double xi = 0.0;
#pragma unroll
          for (int i = 0; i < NM; ++i)
            if (i == t.qoi_index) xi = x[i];
          acc = __dadd_rn(acc, __dmul_rn(sf, xi));
        }
      }
    }
  }
  if (t.x_out >= 0) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (i < n) a.xbuf[t.x_out + i] = x[i];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY) acc = quad_form<NM>(a, Ks, x);
  if (t.qoi_slot >= 0 && t.qoi_mode != MLMCP_QOI_NONE) a.qoi[t.qoi_slot] = acc;
  if (a.iters != nullptr && t.slot >= 0) a.iters[t.slot] = 0;
  if (code != MLMCP_ST_OK) {
    write_status(a.status, t.slot, code, 0, t.tag, t.tag);
    if (a.active != nullptr && t.group >= 0) const_cast<int32_t*>(a.active)[t.group] = 0;
  }
  add_elapsed(a.elapsed, t.slot, t_start);
}

struct DirectCoarseArgs {
  int S, k, m, n;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* M;
  const double* K;
  const double* profile;
  double omega, dt, t0;
  const int64_t* slice_k0;
  const int32_t* slice_steps;
  double* U;
  const double* F;
  double* C;
  int32_t* status;
  int32_t* active;
  int64_t* elapsed;
};

// parareal.py:168-178 (coarse/update sweep of iteration k), one sample per thread
template <int NM>
__global__ void __launch_bounds__(128) direct_coarse_kernel(DirectCoarseArgs c) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= c.S) return;
  const int64_t t_start = global_ns();
  if (c.active[s] == 0) return;
  DirectArgs a{};
  a.n = c.n;
  a.nnz = c.nnz;
  a.row_ptr = c.row_ptr;
  a.col = c.col;
  a.M = c.M;
  a.K = c.K;
  const int n = c.n;
  double m[NM][NM], lu[NM][NM], x[NM], prof[NM], b[NM];
  int piv[NM];
  bool ok;
  factor_task<NM>(a, s, c.dt, m, lu, piv, ok);
  if (!ok) {
    write_status(c.status, s, MLMCP_ST_SINGULAR, 0, c.k, c.k);
    c.active[s] = 0;
    add_elapsed(c.elapsed, s, t_start);
    return;
  }
  const int64_t N = n;
  double* U = c.U + (int64_t)s * (c.m + 1) * N;
  const double* F = c.F + (int64_t)s * (c.m + 1) * N;
  double* C = c.C + (int64_t)s * c.m * N;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    prof[i] = i < n ? c.profile[i] : 0.0;
    if (c.k == 1) {
      x[i] = i < n ? U[i] : 0.0;
    } else {
      x[i] = i < n ? F[(c.k - 1) * N + i] : 0.0;   // freeze U_{k-1} = F_{k-1}
      if (i < n) U[(c.k - 1) * N + i] = x[i];
    }
  }
  for (int sl = c.k; sl < c.m; ++sl) {
    const int steps = c.slice_steps[sl - 1];
    const int64_t k0 = c.slice_k0[sl - 1];
    for (int step = 0; step < steps; ++step) {
      const int64_t g = k0 + step + 1;
      const double sf = sin(__dmul_rn(c.omega, grid_time(c.t0, g, c.dt)));
      rhs<NM>(m, x, prof, c.dt, sf, n, b);
      lu_solve<NM>(lu, piv, n, b);
#pragma unroll
      for (int i = 0; i < NM; ++i) x[i] = b[i];
    }
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      if (i >= n) continue;
      if (c.k == 1) {
        U[sl * N + i] = x[i];
        C[(sl - 1) * N + i] = x[i];
      } else {
        const double c_new = x[i];
        const double un = (F[sl * N + i] + c_new) - C[(sl - 1) * N + i];
        U[sl * N + i] = un;
        C[(sl - 1) * N + i] = c_new;
        x[i] = un;
      }
    }
  }
  if (c.k > 1) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (i < n) U[c.m * N + i] = F[c.m * N + i];
  }
  add_elapsed(c.elapsed, s, t_start);
}

constexpr int kDirectThreads = 128;

}  // namespace

int direct_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* M,
                     const double* K, const double* profile, double omega, double* xbuf,
                     double* qoi, int32_t* iters, int32_t* status, const int32_t* active,
                     int64_t* elapsed, cudaStream_t stream) {
  if (ctx->n > MLMCP_DIRECT_MAX_ROWS) {
    set_error("direct path holds at most MLMCP_DIRECT_MAX_ROWS rows");
    return MLMCP_EINVAL;
  }
  if (n_tasks == 0) return MLMCP_OK;
  DirectArgs a{};
  a.tasks = tasks;
  a.n_tasks = n_tasks;
  a.n = ctx->n;
  a.nnz = ctx->nnz;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.xbuf = xbuf;
  a.qoi = qoi;
  a.iters = iters;
  a.status = status;
  a.active = active;
  a.elapsed = elapsed;
  const unsigned grid = (unsigned)((n_tasks + kDirectThreads - 1) / kDirectThreads);
  direct_propagate_kernel<4><<<grid, kDirectThreads, 0, stream>>>(a);
  MLMCP_LAUNCH_CHECK("direct_propagate_kernel");
  return MLMCP_OK;
}

int direct_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                           const double* profile, double omega, double dt_c, double t0,
                           const int64_t* slice_k0, const int32_t* slice_steps, double* U,
                           const double* F, double* C, int32_t* status, const int32_t* active,
                           int64_t* elapsed, cudaStream_t stream) {
  if (ctx->n > MLMCP_DIRECT_MAX_ROWS) {
    set_error("direct path holds at most MLMCP_DIRECT_MAX_ROWS rows");
    return MLMCP_EINVAL;
  }
  if (S == 0) return MLMCP_OK;
  DirectCoarseArgs c{};
  c.S = S;
  c.k = k;
  c.m = m;
  c.n = ctx->n;
  c.nnz = ctx->nnz;
  c.row_ptr = ctx->row_ptr;
  c.col = ctx->col;
  c.M = M;
  c.K = K;
  c.profile = profile;
  c.omega = omega;
  c.dt = dt_c;
  c.t0 = t0;
  c.slice_k0 = slice_k0;
  c.slice_steps = slice_steps;
  c.U = U;
  c.F = F;
  c.C = C;
  c.status = status;
  c.active = const_cast<int32_t*>(active);
  c.elapsed = elapsed;
  const unsigned grid = (unsigned)((S + kDirectThreads - 1) / kDirectThreads);
  direct_coarse_kernel<4><<<grid, kDirectThreads, 0, stream>>>(c);
  MLMCP_LAUNCH_CHECK("direct_coarse_kernel");
  return MLMCP_OK;
}

}  // namespace mlmcp
