// small_path.cu — SM-resident batched implicit Euler (one CTA per task).
//
// Replaces the per-step dense LU solve of the reference
// (timeint.py:64-75 factorise, :108-110 / :126-127 per-step solve) for
// meshes whose interior system has <= 1024 rows (the 32x32 mesh of configs
// 0/1 has 961).  Each CTA owns one (sample, slice) task for its lifetime:
//   * a thread owns R rows (rows tid, tid+T, ...; T = blockDim.x <= 256): the
//     <= 8 CSR coefficients of A = M + dt*K per row, packed 16-bit smem byte
//     offsets of their columns and D^-1 sit in registers for every step and
//     every PCG iteration (zero HBM traffic for the operator after the first
//     load);
//   * the only shared-memory traffic is the neighbour gather of the SpMV
//     operand (two N-vectors in smem), conflict-free because consecutive
//     lanes own consecutive rows;
//   * PCG is the Chronopoulos-Gear single-reduction variant: one fused block
//     all-reduce (r.u, w.u, r.r) per iteration, two __syncthreads;
//   * few, fat warps (8 warps for 961 rows) keep the per-warp fixed cost of
//     the reductions and the alpha/beta scalar chain small relative to the
//     row work — the loop is issue-bound, not bandwidth-bound;
//   * the QoI (magnetic energy 1/2 x^T K x) is fused into the step loop, so
//     no trajectory is stored unless asked for.
// The Parareal coarse/update sweep (parareal.py:168-178) runs in the same CTA
// model: one CTA per sample walks slices k..M-1 sequentially, the state stays
// in registers between slices.
#include <math.h>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

constexpr int kSmallThreads = 256;

struct SmallShared {
  double* vA;   // gather operand for x (and the energy)
  double* vB;   // gather operand for u
  double* red;  // 2*4*32 block-reduction scratch
  int par;
};

__device__ __forceinline__ double lds_off(const double* base, uint32_t off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + off);
}

// Register state of the R rows of one thread.  Column indices are packed
// 16-bit byte offsets into the shared gather vector (N*8 < 64 KiB).
template <int W, int R>
struct Rows {
  double a[R][W];
  uint32_t cp[R][(W + 1) / 2];
  double dinv[R];

  __device__ __forceinline__ uint32_t off(int r, int j) const {
    const uint32_t w = cp[r][j >> 1];
    return (j & 1) ? (w >> 16) : (w & 0xffffu);
  }

  __device__ __forceinline__ void load(const int32_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col,
                                       const double* __restrict__ Ms,
                                       const double* __restrict__ Ks, double dt, int N) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = threadIdx.x + r * blockDim.x;
      const bool ok = row < N;
      const int q0 = ok ? row_ptr[row] : 0;
      const int len = ok ? row_ptr[row + 1] - q0 : 0;
      double diag = 1.0;
#pragma unroll
      for (int j = 0; j < (W + 1) / 2; ++j) cp[r][j] = 0u;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        uint32_t o;
        if (j < len) {
          const int q = q0 + j;
          const int c = col[q];
          o = (uint32_t)c * 8u;
          a[r][j] = op_entry(__ldg(Ms + q), __ldg(Ks + q), dt);
          if (c == row) diag = a[r][j];
        } else {
          o = ok ? (uint32_t)row * 8u : 0u;
          a[r][j] = 0.0;
        }
        cp[r][j >> 1] |= (j & 1) ? (o << 16) : o;
      }
      dinv[r] = ok ? 1.0 / diag : 0.0;
    }
  }

  // (A v)_row from register coefficients
  __device__ __forceinline__ double spmv(int r, const double* v) const {
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      acc0 = fma(a[r][j], lds_off(v, off(r, j)), acc0);
      if (j + 1 < W) acc1 = fma(a[r][j + 1], lds_off(v, off(r, j + 1)), acc1);
    }
    return acc0 + acc1;
  }

  // (B v)_row for B given by its per-sample CSR values in global memory
  // (M for the right-hand side once per step, K for the energy).
  __device__ __forceinline__ double spmv_csr(int r, const int32_t* __restrict__ row_ptr,
                                             const double* __restrict__ vals,
                                             const double* v) const {
    const int row = threadIdx.x + r * blockDim.x;
    const int q0 = __ldg(row_ptr + row);
    const int len = __ldg(row_ptr + row + 1) - q0;
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      if (j < len) acc0 = fma(__ldg(vals + q0 + j), lds_off(v, off(r, j)), acc0);
      if (j + 1 < W && j + 1 < len)
        acc1 = fma(__ldg(vals + q0 + j + 1), lds_off(v, off(r, j + 1)), acc1);
    }
    return acc0 + acc1;
  }
};

template <int R>
__device__ __forceinline__ bool row_ok(int r, int N) {
  return (int)(threadIdx.x + r * blockDim.x) < N;
}

// 1/2 x^T K x over the block (every thread receives it).  Uses vA.
template <int W, int R>
__device__ __forceinline__ double block_energy(const Rows<W, R>& rw, const double (&x)[R], int N,
                                               const int32_t* __restrict__ row_ptr,
                                               const double* __restrict__ Ks, SmallShared& sh) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) sh.vA[threadIdx.x + r * blockDim.x] = x[r];
  __syncthreads();
  double v[1] = {0.0};
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) v[0] += x[r] * rw.spmv_csr(r, row_ptr, Ks, sh.vA);
  block_allsum<1, kSmallThreads / 32>(v, sh.red, sh.par);
  return 0.5 * v[0];
}

// One implicit-Euler step (M + dt K) x_new = M x + dt*sf*profile by
// Chronopoulos-Gear Jacobi-PCG warm-started at x.  Returns MLMCP_ST_*.
template <int W, int R>
__device__ __forceinline__ int ie_step(const Rows<W, R>& rw, double (&x)[R], int N, double sf,
                                       double dt, const int32_t* __restrict__ row_ptr,
                                       const double* __restrict__ Ms,
                                       const double* __restrict__ profile, double rtol2,
                                       int max_it, SmallShared& sh, int& iters) {
  // b = M x + dt*(sf*prof);  r = b - A x;  u = D r;  w = A u
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) sh.vA[threadIdx.x + r * blockDim.x] = x[r];
  __syncthreads();
  double res[R], u[R], p[R], s[R], w[R];
  double red4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    res[r] = 0.0;
    u[r] = 0.0;
    if (row_ok<R>(r, N)) {
      const int row = threadIdx.x + r * blockDim.x;
      const double mx = rw.spmv_csr(r, row_ptr, Ms, sh.vA);
      const double ax = rw.spmv(r, sh.vA);
      const double b = __dadd_rn(mx, __dmul_rn(dt, __dmul_rn(sf, __ldg(profile + row))));
      res[r] = b - ax;
      u[r] = rw.dinv[r] * res[r];
      red4[3] += b * b;
      sh.vB[row] = u[r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    w[r] = row_ok<R>(r, N) ? rw.spmv(r, sh.vB) : 0.0;
    red4[0] += res[r] * u[r];
    red4[1] += w[r] * u[r];
    red4[2] += res[r] * res[r];
  }
  block_allsum<4, kSmallThreads / 32>(red4, sh.red, sh.par);
  double gamma = red4[0];
  double delta = red4[1];
  double rho = red4[2];
  const double bnorm2 = red4[3];
  if (bnorm2 == 0.0) {  // b == 0 exactly: the solution is 0
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = 0.0;
    return MLMCP_ST_OK;
  }
  const double tol2 = rtol2 * bnorm2;
  if (rho <= tol2) return MLMCP_ST_OK;
  if (!isfinite(rho)) return MLMCP_ST_NONFINITE;
  if (!(delta > 0.0)) return MLMCP_ST_BREAKDOWN;
  double alpha = gamma / delta;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    p[r] = u[r];
    s[r] = w[r];
    x[r] = fma(alpha, p[r], x[r]);
    res[r] = fma(-alpha, s[r], res[r]);
  }
  int it = 1;
  for (;;) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      u[r] = rw.dinv[r] * res[r];              // 0 on padding rows (dinv = 0)
      sh.vB[threadIdx.x + r * blockDim.x] = u[r];  // vB is padded to R*blockDim
    }
    __syncthreads();
    double red3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      w[r] = rw.spmv(r, sh.vB);                // a = 0 on padding rows
      red3[0] += res[r] * u[r];
      red3[1] += w[r] * u[r];
      red3[2] += res[r] * res[r];
    }
    block_allsum<3, kSmallThreads / 32>(red3, sh.red, sh.par);
    const double gnew = red3[0];
    delta = red3[1];
    rho = red3[2];
    if (rho <= tol2) break;
    if (!isfinite(rho)) { iters += it; return MLMCP_ST_NONFINITE; }
    if (it >= max_it) { iters += it; return MLMCP_ST_NOCONV; }
    const double beta = gnew / gamma;
    const double den = delta - beta * gnew / alpha;
    if (!(den > 0.0)) { iters += it; return MLMCP_ST_BREAKDOWN; }
    alpha = gnew / den;
    gamma = gnew;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      p[r] = fma(beta, p[r], u[r]);
      s[r] = fma(beta, s[r], w[r]);
      x[r] = fma(alpha, p[r], x[r]);
      res[r] = fma(-alpha, s[r], res[r]);
    }
    ++it;
  }
  iters += it;
  return MLMCP_ST_OK;
}

struct SmallArgs {
  const mlmcp_task* tasks;
  int n_tasks;
  int N;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* M;
  const double* K;
  const double* profile;
  double omega;
  double rtol2;
  int max_it;
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  int32_t* active;
};

template <int W, int R>
__global__ void __launch_bounds__(kSmallThreads, 1) small_propagate_kernel(SmallArgs a) {
  extern __shared__ double smem[];
  const mlmcp_task t = a.tasks[blockIdx.x];
  {
    // another CTA of the same group may clear active[] concurrently (on a
    // failure): decide once per block so the barriers below never diverge
    __shared__ int skip;
    if (threadIdx.x == 0)
      skip = (a.active != nullptr && t.group >= 0 && a.active[t.group] == 0) ? 1 : 0;
    __syncthreads();
    if (skip) return;
  }
  const int padN = R * blockDim.x;
  SmallShared sh{smem, smem + padN, smem + 2 * padN, 0};
  const double* Ms = a.M + (int64_t)t.sample * a.nnz;
  const double* Ks = a.K + (int64_t)t.sample * a.nnz;
  Rows<W, R> rw;
  rw.load(a.row_ptr, a.col, Ms, Ks, t.dt, a.N);
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = threadIdx.x + r * blockDim.x;
    x[r] = row_ok<R>(r, a.N) ? a.xbuf[t.x_in + row] : 0.0;
    if (t.traj >= 0 && row_ok<R>(r, a.N)) a.xbuf[t.traj + row] = x[r];
  }
  int iters = 0;
  int code = MLMCP_ST_OK;
  int fail_step = 0;
  double acc = 0.0;
  for (int step = 0; step < t.n_steps; ++step) {
    const int64_t g = t.k0 + step + 1;
    const double sf = sin(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)));
    code = ie_step(rw, x, a.N, sf, t.dt, a.row_ptr, Ms, a.profile, a.rtol2, a.max_it, sh, iters);
    if (code != MLMCP_ST_OK) { fail_step = step; break; }
    if (t.traj >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (row_ok<R>(r, a.N))
          a.xbuf[t.traj + (int64_t)(step + 1) * a.N + threadIdx.x + r * blockDim.x] = x[r];
    }
    if (t.qoi_mode == MLMCP_QOI_SUM_ENERGY && g > t.qoi_from)
      acc += block_energy(rw, x, a.N, a.row_ptr, Ks, sh);
  }
  if (t.x_out >= 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (row_ok<R>(r, a.N)) a.xbuf[t.x_out + threadIdx.x + r * blockDim.x] = x[r];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY && t.qoi_slot >= 0)
    acc = block_energy(rw, x, a.N, a.row_ptr, Ks, sh);
  if (threadIdx.x == 0) {
    if (t.qoi_slot >= 0 && t.qoi_mode != MLMCP_QOI_NONE) a.qoi[t.qoi_slot] = acc;
    if (a.iters != nullptr && t.slot >= 0) a.iters[t.slot] = iters;
    if (code != MLMCP_ST_OK) {
      write_status(a.status, t.slot, code, fail_step, t.tag, t.tag);
      if (a.active != nullptr && t.group >= 0) a.active[t.group] = 0;
    }
  }
}

struct CoarseArgs {
  int S, k, m, N;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* M;
  const double* K;
  const double* profile;
  double omega, dt, t0, rtol2;
  int max_it;
  const int64_t* slice_k0;
  const int32_t* slice_steps;
  double* U;
  const double* F;
  double* C;
  int32_t* iters;
  int32_t* status;
  int32_t* active;
};

// parareal.py:168-178 for one sample per CTA.
template <int W, int R>
__global__ void __launch_bounds__(kSmallThreads, 1) small_coarse_kernel(CoarseArgs a) {
  extern __shared__ double smem[];
  const int s = blockIdx.x;
  if (a.active[s] == 0) return;
  const int padN = R * blockDim.x;
  SmallShared sh{smem, smem + padN, smem + 2 * padN, 0};
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  Rows<W, R> rw;
  rw.load(a.row_ptr, a.col, Ms, Ks, a.dt, a.N);
  const int64_t N = a.N;
  double* U = a.U + (int64_t)s * (a.m + 1) * N;
  const double* F = a.F + (int64_t)s * (a.m + 1) * N;
  double* C = a.C + (int64_t)s * a.m * N;
  int iters = 0;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = threadIdx.x + r * blockDim.x;
    const bool ok = row_ok<R>(r, a.N);
    if (a.k == 1) {
      x[r] = ok ? U[i] : 0.0;
    } else {
      x[r] = ok ? F[(a.k - 1) * N + i] : 0.0;  // freeze U_{k-1} = F_{k-1}
      if (ok) U[(a.k - 1) * N + i] = x[r];
    }
  }
  for (int n = a.k; n < a.m; ++n) {
    const int steps = a.slice_steps[n - 1];
    const int64_t k0 = a.slice_k0[n - 1];
    for (int step = 0; step < steps; ++step) {
      const int64_t g = k0 + step + 1;
      const double sf = sin(__dmul_rn(a.omega, grid_time(a.t0, g, a.dt)));
      const int code =
          ie_step(rw, x, a.N, sf, a.dt, a.row_ptr, Ms, a.profile, a.rtol2, a.max_it, sh, iters);
      if (code != MLMCP_ST_OK) {
        if (threadIdx.x == 0) {
          write_status(a.status, s, code, step, n, a.k);
          a.active[s] = 0;
          if (a.iters != nullptr) a.iters[s] += iters;
        }
        return;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = threadIdx.x + r * blockDim.x;
      if (!row_ok<R>(r, a.N)) continue;
      if (a.k == 1) {
        U[n * N + i] = x[r];
        C[(n - 1) * N + i] = x[r];
      } else {
        const double c_new = x[r];
        const double un = (F[n * N + i] + c_new) - C[(n - 1) * N + i];
        U[n * N + i] = un;
        C[(n - 1) * N + i] = c_new;
        x[r] = un;
      }
    }
  }
  if (a.k > 1) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = threadIdx.x + r * blockDim.x;
      if (row_ok<R>(r, a.N)) U[a.m * N + i] = F[a.m * N + i];
    }
  }
  if (threadIdx.x == 0 && a.iters != nullptr) a.iters[s] += iters;
  (void)Ks;
}

inline int rows_per_thread(int N) {
  if (N <= kSmallThreads) return 1;
  if (N <= 2 * kSmallThreads) return 2;
  return 4;
}
inline int block_threads(int N, int R) { return ((N + R - 1) / R + 31) / 32 * 32; }
inline size_t small_smem(int padN) { return (size_t)(2 * padN + 2 * 4 * 32) * sizeof(double); }

template <template <int, int> class Launch, typename Args>
int dispatch(int W, int N, const Args& a, unsigned grid, cudaStream_t stream) {
  const int R = rows_per_thread(N);
  const int nt = block_threads(N, R);
  const size_t smem = small_smem(R * nt);
#define MLMCP_CASE_R(WW, RR) \
  if (W == WW && R == RR) return Launch<WW, RR>::run(a, grid, nt, smem, stream);
#define MLMCP_CASE(WW) MLMCP_CASE_R(WW, 1) MLMCP_CASE_R(WW, 2) MLMCP_CASE_R(WW, 4)
  MLMCP_CASE(1) MLMCP_CASE(2) MLMCP_CASE(3) MLMCP_CASE(4)
  MLMCP_CASE(5) MLMCP_CASE(6) MLMCP_CASE(7) MLMCP_CASE(8)
#undef MLMCP_CASE
#undef MLMCP_CASE_R
  set_error("unsupported row width");
  return MLMCP_EINVAL;
}

template <int W, int R>
struct LaunchPropagate {
  static int run(const SmallArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    small_propagate_kernel<W, R><<<grid, nt, smem, st>>>(a);
    MLMCP_LAUNCH_CHECK("small_propagate_kernel");
    return MLMCP_OK;
  }
};

template <int W, int R>
struct LaunchCoarse {
  static int run(const CoarseArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    small_coarse_kernel<W, R><<<grid, nt, smem, st>>>(a);
    MLMCP_LAUNCH_CHECK("small_coarse_kernel");
    return MLMCP_OK;
  }
};

}  // namespace

int small_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* M,
                    const double* K, const double* profile, double omega, double rtol,
                    int max_it, double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                    const int32_t* active, cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  SmallArgs a{tasks, n_tasks, ctx->n, ctx->nnz, ctx->row_ptr, ctx->col, M, K, profile,
              omega, rtol * rtol, max_it, xbuf, qoi, iters, status,
              const_cast<int32_t*>(active)};
  return dispatch<LaunchPropagate>(ctx->max_row_nnz, ctx->n, a, (unsigned)n_tasks, stream);
}

int small_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                          const double* profile, double omega, double dt_c, double t0,
                          const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                          int max_it, double* U, const double* F, double* C, int32_t* iters,
                          int32_t* status, const int32_t* active, cudaStream_t stream) {
  if (S == 0) return MLMCP_OK;
  CoarseArgs a{S, k, m, ctx->n, ctx->nnz, ctx->row_ptr, ctx->col, M, K, profile, omega, dt_c,
               t0, rtol * rtol, max_it, slice_k0, slice_steps, U, F, C, iters, status,
               const_cast<int32_t*>(active)};
  return dispatch<LaunchCoarse>(ctx->max_row_nnz, ctx->n, a, (unsigned)S, stream);
}

}  // namespace mlmcp
