// small_path.cu — SM-resident batched implicit Euler (one CTA per task).
//
// Replaces the per-step dense LU solve of the reference
// (timeint.py:64-75 factorise, :108-110 / :126-127 per-step solve) for
// meshes whose interior system has <= 1024 rows (the 32x32 mesh of configs
// 0/1 has 961).  Each CTA owns one (sample, slice) task for its lifetime:
//   * a thread owns R rows (rows tid, tid+256, ...; 256 threads per CTA): the
//     <= 8 coefficients of A = M + dt*K per row and D^-1 sit in registers for
//     every step and every PCG iteration (no HBM traffic for the operator
//     after the first load);
//   * column addressing has two policies:
//       STENCIL  the pattern is a uniform-offset stencil (every col - row in a
//                set of <= 8 offsets: the structured 7-point FE mesh, banded
//                models) -> neighbour j of row i is v[i + off_j], off_j
//                block-uniform; zero-padded smem vectors absorb the missing
//                boundary neighbours (their coefficients are 0).  No per-row
//                column registers: two CTAs fit one SM.
//       CSR      generic pattern -> packed 16-bit smem byte offsets per entry.
//   * the only shared-memory traffic is the neighbour gather of the SpMV
//     operand, conflict-free because consecutive lanes own consecutive rows;
//   * PCG is the Chronopoulos-Gear single-reduction variant: one fused block
//     all-reduce (r.u, w.u, r.r) per iteration, two __syncthreads; the
//     alpha/beta recurrence needs one reciprocal on the critical path (1/gamma
//     and 1/alpha for the next iteration are formed off the critical path);
//   * the cross-warp stage of the reduction is a broadcast smem read of the
//     <= 8 warp partials + a fixed tree (no second butterfly);
//   * the QoI (magnetic energy 1/2 x^T K x) is fused into the step loop, so
//     no trajectory is stored unless asked for.
// The Parareal coarse/update sweep (parareal.py:168-178) runs in the same CTA
// model: one CTA per sample walks slices k..M-1 sequentially, the state stays
// in registers between slices.
#include <math.h>
#include <stdlib.h>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

constexpr int kSmallThreads = 256;
constexpr int kMaxWarps = kSmallThreads / 32;

struct StencilArgs {
  int off[kMaxNz];       // sorted offsets (col - row)
  int off8[kMaxNz];      // the same in bytes
  const int32_t* pos;    // [W][N] CSR position of slot j of row i, or -1
};

struct SmallShared {
  double* vA;   // gather operand for x (and the energy); row 0 at vA[0]
  double* vB;   // gather operand for u
  double* red;  // [2][kMaxWarps][4]
  int par;
};

// Block all-reduce of NV <= 4 doubles.  Butterfly inside each warp, then every
// thread reads the <= 8 warp partials (broadcast) and sums them in a fixed
// tree: bitwise identical totals in all threads, deterministic.
template <int NV>
__device__ __forceinline__ void cta_allsum(double (&v)[NV], SmallShared& sh) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  double* buf = sh.red + sh.par * (kMaxWarps * 4);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) buf[warp * 4 + k] = v[k];
  }
  __syncthreads();
  // fixed pairwise tree ((w0+w1)+(w2+w3))+((w4+w5)+(w6+w7)), streamed so that
  // only a few partials are live at a time (register pressure)
  auto ld = [&](int w, double (&o)[NV]) {
    if (w < nwarps) {
      const double2 lo = *reinterpret_cast<const double2*>(buf + w * 4);
      o[0] = lo.x;
      if (NV > 1) o[1 % NV] = lo.y;
      if (NV > 2) {
        const double2 hi = *reinterpret_cast<const double2*>(buf + w * 4 + 2);
        o[2 % NV] = hi.x;
        if (NV > 3) o[3 % NV] = hi.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) o[k] = 0.0;
    }
  };
  static_assert(kMaxWarps == 8, "tree below is written for 8 warps");
  double q0[NV], q1[NV], h0[NV], h1[NV];
  ld(0, q0); ld(1, q1);
#pragma unroll
  for (int k = 0; k < NV; ++k) h0[k] = q0[k] + q1[k];
  ld(2, q0); ld(3, q1);
#pragma unroll
  for (int k = 0; k < NV; ++k) h0[k] = h0[k] + (q0[k] + q1[k]);
  ld(4, q0); ld(5, q1);
#pragma unroll
  for (int k = 0; k < NV; ++k) h1[k] = q0[k] + q1[k];
  ld(6, q0); ld(7, q1);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = h0[k] + (h1[k] + (q0[k] + q1[k]));
  sh.par ^= 1;
}

__device__ __forceinline__ double lds_off(const double* base, uint32_t off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + off);
}

// Every SM-resident CTA has exactly kSmallThreads threads (rows beyond N are
// zero padding), so row addresses fold into compile-time immediates.
template <int R>
__device__ __forceinline__ int row_of(int r) {
  return threadIdx.x + r * kSmallThreads;
}

template <int R>
__device__ __forceinline__ bool row_ok(int r, int N) {
  return row_of<R>(r) < N;
}

// Register state of the R rows of one thread.
template <int W, int R, bool ST>
struct Rows {
  double a[R][W];
  uint32_t cp[ST ? 1 : R][ST ? 1 : (W + 1) / 2];  // CSR: packed smem byte offsets
  double dinv[R];

  __device__ __forceinline__ uint32_t off(int r, int j) const {
    const uint32_t w = cp[ST ? 0 : r][ST ? 0 : (j >> 1)];
    return (j & 1) ? (w >> 16) : (w & 0xffffu);
  }

  __device__ __forceinline__ void load(const int32_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col, const StencilArgs& st,
                                       const double* __restrict__ Ms,
                                       const double* __restrict__ Ks, double dt, int N) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = row_of<R>(r);
      const bool ok = row < N;
      double diag = 1.0;
      if (ST) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int q = ok ? st.pos[j * N + row] : -1;
          a[r][j] = q >= 0 ? op_entry(__ldg(Ms + q), __ldg(Ks + q), dt) : 0.0;
          if (st.off[j] == 0 && q >= 0) diag = a[r][j];
        }
      } else {
        const int q0 = ok ? row_ptr[row] : 0;
        const int len = ok ? row_ptr[row + 1] - q0 : 0;
#pragma unroll
        for (int j = 0; j < (W + 1) / 2; ++j) cp[ST ? 0 : r][ST ? 0 : j] = 0u;
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
          cp[ST ? 0 : r][ST ? 0 : (j >> 1)] |= (j & 1) ? (o << 16) : o;
        }
      }
      dinv[r] = ok ? 1.0 / diag : 0.0;
    }
  }

  __device__ __forceinline__ double gather(int r, int j, const double* v,
                                           const StencilArgs& st) const {
    if (ST) return lds_off(v + row_of<R>(r), (uint32_t)st.off8[j]);
    return lds_off(v, off(r, j));
  }

  // (A v)_row from register coefficients
  __device__ __forceinline__ double spmv(int r, const double* v, const StencilArgs& st) const {
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      acc0 = fma(a[r][j], gather(r, j, v, st), acc0);
      if (j + 1 < W) acc1 = fma(a[r][j + 1], gather(r, j + 1, v, st), acc1);
    }
    return acc0 + acc1;
  }

  // (B v)_row for B given by per-sample CSR values in global memory (M for the
  // right-hand side once per step, K for the energy).  Only for rows < N.
  __device__ __forceinline__ double spmv_csr(int r, const int32_t* __restrict__ row_ptr,
                                             const StencilArgs& st, int N,
                                             const double* __restrict__ vals,
                                             const double* v) const {
    const int row = row_of<R>(r);
    double acc0 = 0.0, acc1 = 0.0;
    if (ST) {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int q = __ldg(st.pos + j * N + row);
        const double t = q >= 0 ? __ldg(vals + q) * v[row + st.off[j]] : 0.0;
        if (j & 1) acc1 += t;
        else acc0 += t;
      }
    } else {
      const int q0 = __ldg(row_ptr + row);
      const int len = __ldg(row_ptr + row + 1) - q0;
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        if (j < len) acc0 = fma(__ldg(vals + q0 + j), lds_off(v, off(r, j)), acc0);
        if (j + 1 < W && j + 1 < len)
          acc1 = fma(__ldg(vals + q0 + j + 1), lds_off(v, off(r, j + 1)), acc1);
      }
    }
    return acc0 + acc1;
  }
};

// 1/2 x^T K x over the block (every thread receives it).  Uses vA.
template <int W, int R, bool ST>
__device__ __forceinline__ double block_energy(const Rows<W, R, ST>& rw, const double (&x)[R],
                                               int N, const int32_t* __restrict__ row_ptr,
                                               const StencilArgs& st,
                                               const double* __restrict__ Ks, SmallShared& sh) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) sh.vA[row_of<R>(r)] = x[r];
  __syncthreads();
  double v[1] = {0.0};
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) v[0] += x[r] * rw.spmv_csr(r, row_ptr, st, N, Ks, sh.vA);
  cta_allsum<1>(v, sh);
  return 0.5 * v[0];
}

// One implicit-Euler step (M + dt K) x_new = M x + dt*sf*profile by
// Chronopoulos-Gear Jacobi-PCG warm-started at x.  Returns MLMCP_ST_*.
template <int W, int R, bool ST>
__device__ __forceinline__ int ie_step(const Rows<W, R, ST>& rw, double (&x)[R], int N,
                                       double sf, double dt, const int32_t* __restrict__ row_ptr,
                                       const StencilArgs& st, const double* __restrict__ Ms,
                                       const double* __restrict__ profile, double rtol2,
                                       int max_it, SmallShared& sh, int& iters) {
  // b = M x + dt*(sf*prof);  r = b - A x;  u = D r;  w = A u
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (row_ok<R>(r, N)) sh.vA[row_of<R>(r)] = x[r];
  __syncthreads();
  double res[R], u[R], p[R], s[R], w[R];
  double red4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    res[r] = 0.0;
    u[r] = 0.0;
    if (row_ok<R>(r, N)) {
      const int row = row_of<R>(r);
      const double mx = rw.spmv_csr(r, row_ptr, st, N, Ms, sh.vA);
      const double ax = rw.spmv(r, sh.vA, st);
      const double b = __dadd_rn(mx, __dmul_rn(dt, __dmul_rn(sf, __ldg(profile + row))));
      res[r] = b - ax;
      u[r] = rw.dinv[r] * res[r];
      red4[3] += b * b;
    }
    sh.vB[row_of<R>(r)] = u[r];            // vB is padded to R*256 rows
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    w[r] = rw.spmv(r, sh.vB, st);          // a = 0 on padding rows
    red4[0] += res[r] * u[r];
    red4[1] += w[r] * u[r];
    red4[2] += res[r] * res[r];
  }
  cta_allsum<4>(red4, sh);
  const double gamma = red4[0];
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
  double alpha = gamma * fast_rcp(delta);
  double inv_g = fast_rcp(gamma);
  double c = inv_g * (delta * inv_g);      // 1/(gamma * alpha) = delta / gamma^2
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
      u[r] = rw.dinv[r] * res[r];          // 0 on padding rows (dinv = 0)
      sh.vB[row_of<R>(r)] = u[r];
    }
    __syncthreads();
    double red3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      w[r] = rw.spmv(r, sh.vB, st);
      red3[0] += res[r] * u[r];
      red3[1] += w[r] * u[r];
      red3[2] += res[r] * res[r];
    }
    cta_allsum<3>(red3, sh);
    const double gnew = red3[0];
    delta = red3[1];
    rho = red3[2];
    if (rho <= tol2) break;
    if (!isfinite(rho)) { iters += it; return MLMCP_ST_NONFINITE; }
    if (it >= max_it) { iters += it; return MLMCP_ST_NOCONV; }
    // beta = gnew/gamma, alpha = gnew / (delta - beta*gnew/alpha)
    const double beta = gnew * inv_g;
    const double den = fma(-(gnew * gnew), c, delta);
    if (!(den > 0.0)) { iters += it; return MLMCP_ST_BREAKDOWN; }
    const double rden = fast_rcp(den);
    alpha = gnew * rden;
    inv_g = fast_rcp(gnew);                // off the critical path (next iteration)
    c = inv_g * (den * inv_g);             // 1/(gnew*alpha)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      p[r] = fma(beta, p[r], rw.dinv[r] * res[r]);   // u recomputed: fewer live registers
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
  StencilArgs st;
  int pad;               // zero rows before row 0 / after the last padded row
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

// Carve and zero the padded smem vectors.
template <int R>
__device__ __forceinline__ SmallShared setup_shared(double* smem, int pad) {
  const int len = pad + R * kSmallThreads + pad;
  for (int i = threadIdx.x; i < 2 * len; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();
  return SmallShared{smem + pad, smem + len + pad, smem + 2 * len, 0};
}

template <int W, int R, bool ST, int OCC>
__global__ void __launch_bounds__(kSmallThreads, OCC) small_propagate_kernel(SmallArgs a) {
  extern __shared__ __align__(16) double smem[];
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
  SmallShared sh = setup_shared<R>(smem, a.pad);
  const double* Ms = a.M + (int64_t)t.sample * a.nnz;
  const double* Ks = a.K + (int64_t)t.sample * a.nnz;
  Rows<W, R, ST> rw;
  rw.load(a.row_ptr, a.col, a.st, Ms, Ks, t.dt, a.N);
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int row = row_of<R>(r);
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
    code = ie_step(rw, x, a.N, sf, t.dt, a.row_ptr, a.st, Ms, a.profile, a.rtol2, a.max_it, sh,
                   iters);
    if (code != MLMCP_ST_OK) { fail_step = step; break; }
    if (t.traj >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (row_ok<R>(r, a.N)) a.xbuf[t.traj + (int64_t)(step + 1) * a.N + row_of<R>(r)] = x[r];
    }
    if (t.qoi_mode == MLMCP_QOI_SUM_ENERGY && g > t.qoi_from)
      acc += block_energy(rw, x, a.N, a.row_ptr, a.st, Ks, sh);
  }
  if (t.x_out >= 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (row_ok<R>(r, a.N)) a.xbuf[t.x_out + row_of<R>(r)] = x[r];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY && t.qoi_slot >= 0)
    acc = block_energy(rw, x, a.N, a.row_ptr, a.st, Ks, sh);
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
  StencilArgs st;
  int pad;
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
template <int W, int R, bool ST, int OCC>
__global__ void __launch_bounds__(kSmallThreads, OCC) small_coarse_kernel(CoarseArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int s = blockIdx.x;
  if (a.active[s] == 0) return;
  SmallShared sh = setup_shared<R>(smem, a.pad);
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  Rows<W, R, ST> rw;
  rw.load(a.row_ptr, a.col, a.st, Ms, Ks, a.dt, a.N);
  const int64_t N = a.N;
  double* U = a.U + (int64_t)s * (a.m + 1) * N;
  const double* F = a.F + (int64_t)s * (a.m + 1) * N;
  double* C = a.C + (int64_t)s * a.m * N;
  int iters = 0;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = row_of<R>(r);
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
      const int code = ie_step(rw, x, a.N, sf, a.dt, a.row_ptr, a.st, Ms, a.profile, a.rtol2,
                               a.max_it, sh, iters);
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
      const int i = row_of<R>(r);
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
      const int i = row_of<R>(r);
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
inline int block_threads(int, int) { return kSmallThreads; }
inline size_t small_smem(int padN, int pad) {
  return (size_t)(2 * (padN + 2 * pad) + 2 * kMaxWarps * 4) * sizeof(double);
}

template <template <int, int, bool, int> class Launch, typename Args>
int dispatch(const Ctx* ctx, Args& a, unsigned grid, cudaStream_t stream) {
  const int N = ctx->n;
  const int R = rows_per_thread(N);
  const int nt = block_threads(N, R);
  const bool st = ctx->stencil_w > 0;
  const int W = st ? ctx->stencil_w : ctx->max_row_nnz;
  a.pad = st ? ctx->stencil_pad : 0;
  if (st) {
    for (int k = 0; k < kMaxNz; ++k) {
      a.st.off[k] = k < W ? ctx->stencil_off[k] : 0;
      a.st.off8[k] = a.st.off[k] * 8;
    }
    a.st.pos = ctx->stencil_pos;
  } else {
    a.st.pos = nullptr;
  }
  const size_t smem = small_smem(R * nt, a.pad);
  if (smem > 200 * 1024) {
    set_error("SM-resident path: shared-memory footprint too large for this pattern");
    return MLMCP_EINVAL;
  }
  // two CTAs per SM for the stencil path (128 registers per thread) unless
  // MLMCP_SMALL_OCC=1 asks for one (255 registers, no spills)
  static const int occ = [] {
    const char* e = getenv("MLMCP_SMALL_OCC");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
#define MLMCP_CASE_R(WW, RR)                                                       \
  if (W == WW && R == RR) {                                                        \
    if (!st) return Launch<WW, RR, false, 1>::run(a, grid, nt, smem, stream);      \
    if (RR == 4 && occ == 2) return Launch<WW, RR, true, 2>::run(a, grid, nt, smem, stream); \
    return Launch<WW, RR, true, 1>::run(a, grid, nt, smem, stream);                \
  }
#define MLMCP_CASE(WW) MLMCP_CASE_R(WW, 1) MLMCP_CASE_R(WW, 2) MLMCP_CASE_R(WW, 4)
  MLMCP_CASE(1) MLMCP_CASE(2) MLMCP_CASE(3) MLMCP_CASE(4)
  MLMCP_CASE(5) MLMCP_CASE(6) MLMCP_CASE(7) MLMCP_CASE(8)
#undef MLMCP_CASE
#undef MLMCP_CASE_R
  set_error("unsupported row width");
  return MLMCP_EINVAL;
}

template <int W, int R, bool ST, int OCC>
struct LaunchPropagate {
  static int run(const SmallArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(small_propagate_kernel<W, R, ST, OCC>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    small_propagate_kernel<W, R, ST, OCC><<<grid, nt, smem, st>>>(a);
    MLMCP_LAUNCH_CHECK("small_propagate_kernel");
    return MLMCP_OK;
  }
};

template <int W, int R, bool ST, int OCC>
struct LaunchCoarse {
  static int run(const CoarseArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(small_coarse_kernel<W, R, ST, OCC>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    small_coarse_kernel<W, R, ST, OCC><<<grid, nt, smem, st>>>(a);
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
  SmallArgs a{};
  a.tasks = tasks;
  a.n_tasks = n_tasks;
  a.N = ctx->n;
  a.nnz = ctx->nnz;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.xbuf = xbuf;
  a.qoi = qoi;
  a.iters = iters;
  a.status = status;
  a.active = const_cast<int32_t*>(active);
  return dispatch<LaunchPropagate>(ctx, a, (unsigned)n_tasks, stream);
}

int small_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                          const double* profile, double omega, double dt_c, double t0,
                          const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                          int max_it, double* U, const double* F, double* C, int32_t* iters,
                          int32_t* status, const int32_t* active, cudaStream_t stream) {
  if (S == 0) return MLMCP_OK;
  CoarseArgs a{};
  a.S = S;
  a.k = k;
  a.m = m;
  a.N = ctx->n;
  a.nnz = ctx->nnz;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.dt = dt_c;
  a.t0 = t0;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.slice_k0 = slice_k0;
  a.slice_steps = slice_steps;
  a.U = U;
  a.F = F;
  a.C = C;
  a.iters = iters;
  a.status = status;
  a.active = const_cast<int32_t*>(active);
  return dispatch<LaunchCoarse>(ctx, a, (unsigned)S, stream);
}

}  // namespace mlmcp
