// stream_path.cu — HBM-streaming batched implicit Euler for meshes whose
// interior system does not fit one SM (128^2 .. 512^2: configs 2, 3, 4).
//
// Same numerical method and step semantics as small_path.cu (reference:
// timeint.py:88-128: extrapolated initial guesses, Jacobi-weighted stopping
// rule), but every PCG iteration is two grid-wide launches over all live
// (task, row-block) pairs:
//   K_spmv   w = A (D^-1 r) with the operator in a per-sample ELL layout
//            [S][W][N] (coalesced, built once per call from the CSR M/K
//            values), partial (r.u, w.u, r.r) per block; the last block of a
//            task (arrival counter) reduces the partials in fixed order and
//            computes alpha/beta, the convergence test and the failure codes.
//   K_update p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s.
// Per-task scalars live in the workspace; converged tasks skip their blocks.
// The host loop launches chunks of iterations sized by the previous step's
// count and reads one pinned 8-byte counter per chunk (the only host sync).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

constexpr int kThreads = 256;

enum : int { ST_IDLE = 0, ST_RUN = 1, ST_DONE = 2, ST_ZERO = 3 };

// task scalar layout (doubles)
enum : int { D_BB = 0, D_GAMMA, D_ALPHA, D_BETA, D_ACC, D_SF, kTD };
// task int layout
enum : int { I_STATE = 0, I_IT_STEP, I_IT_TOTAL, I_CODE, I_FAILSTEP, I_FIRST, kTI };

constexpr int kRingS = 8;   // past states a_{n-1..n-8} (extrapolation order <= 7)

// extrapolation weights: a_{n+1} ~ sum_j c[p][j] a_{n-j}, c[p][j] = (-1)^j C(p+1, j+1)
__constant__ double c_extrap[8][8] = {
    {1, 0, 0, 0, 0, 0, 0, 0},
    {2, -1, 0, 0, 0, 0, 0, 0},
    {3, -3, 1, 0, 0, 0, 0, 0},
    {4, -6, 4, -1, 0, 0, 0, 0},
    {5, -10, 10, -5, 1, 0, 0, 0},
    {6, -15, 20, -15, 6, -1, 0, 0},
    {7, -21, 35, -35, 21, -7, 1, 0},
    {8, -28, 56, -70, 56, -28, 8, -1}};
// least-squares degree-6 fit through y_n .. y_{n-7}, extrapolated one step:
// with the steady-state predictor (rtol 1e-14) it beats the exact order-7
// polynomial (sum |w| 69 vs 255), numpy model of config 2: 4.4 -> 3.6
// iterations per step
__constant__ int c_ls_on = 1;   // MLMCP_LSGUESS=0 disables (A/B)
__constant__ double c_ls68[8] = {49.0 / 8, -119.0 / 8, 133.0 / 8, -35.0 / 8,
                                 -77.0 / 8, 91.0 / 8, -41.0 / 8, 7.0 / 8};

struct Work {
  double* ring;    // [kRingS][T][N]
  double* A;       // [S][W][N]
  double* dinv;    // [S][N]
  double* X;       // [T][N]
  double* R;
  double* P;
  double* Sv;
  double* Wv;
  double* R1;      // tile path: second buffers of r, w, s (ping-pong by iteration parity)
  double* W1;
  double* S1;
  double* ctab;    // region mode: [T][15][rC] per-task class stencils (build_class_table)
  double* partial; // [T][nblk][4]
  double* td;      // [T][kTD]
  int32_t* ti;     // [T][kTI]
  int32_t* arrive; // [T]
  int32_t* counters;  // [0] live, [1] done
};

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t off[17];
  size_t total;
};

Layout make_layout(const Ctx* ctx, int T, int S) {
  // operator slots: ELL width, or the stencil width for the cooperative path
  const size_t N = ctx->n, W = std::max(ctx->max_row_nnz, ctx->stencil_w), T_ = T, S_ = S;
  const size_t nblk = (N + kThreads - 1) / kThreads;
  size_t sizes[17] = {S_ * std::max(W, (size_t)8) * N * 8, S_ * N * 8, T_ * N * 8, T_ * N * 8, T_ * N * 8,
                      T_ * N * 8,     T_ * N * 8, T_ * nblk * 4 * 8, T_ * kTD * 8,
                      T_ * kTI * 4,   T_ * 4,     64, kRingS * T_ * N * 8,
                      T_ * N * 8,     T_ * N * 8, T_ * N * 8, T_ * 15 * (size_t)ctx->rC * 8};
  Layout L;
  size_t o = 0;
  for (int i = 0; i < 17; ++i) {
    L.off[i] = o;
    o += align_up(sizes[i]);
  }
  L.total = o + 256;   // bulk row copies may read up to one element past the last vector
  return L;
}

Work carve(void* ws, const Layout& L) {
  char* b = static_cast<char*>(ws);
  Work w;
  w.A = reinterpret_cast<double*>(b + L.off[0]);
  w.dinv = reinterpret_cast<double*>(b + L.off[1]);
  w.X = reinterpret_cast<double*>(b + L.off[2]);
  w.R = reinterpret_cast<double*>(b + L.off[3]);
  w.P = reinterpret_cast<double*>(b + L.off[4]);
  w.Sv = reinterpret_cast<double*>(b + L.off[5]);
  w.Wv = reinterpret_cast<double*>(b + L.off[6]);
  w.partial = reinterpret_cast<double*>(b + L.off[7]);
  w.td = reinterpret_cast<double*>(b + L.off[8]);
  w.ti = reinterpret_cast<int32_t*>(b + L.off[9]);
  w.arrive = reinterpret_cast<int32_t*>(b + L.off[10]);
  w.counters = reinterpret_cast<int32_t*>(b + L.off[11]);
  w.ring = reinterpret_cast<double*>(b + L.off[12]);
  w.R1 = reinterpret_cast<double*>(b + L.off[13]);
  w.W1 = reinterpret_cast<double*>(b + L.off[14]);
  w.S1 = reinterpret_cast<double*>(b + L.off[15]);
  w.ctab = reinterpret_cast<double*>(b + L.off[16]);
  return w;
}

struct SArgs {
  int T, S, N, W, nblk;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* ell_col;
  const int32_t* ell_pos;
  const mlmcp_task* tasks;
  const double* M;
  const double* K;
  const double* profile;
  double omega, rtol2;
  int max_it;
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  int32_t* active;
  const double* xss;   // [slots][2][N] periodic steady states (task.ss_slot) or null
  // tile path (structured wd x gh grid): operator [S][4][N] (C, E, N, NE) in w.A
  int tile;            // 1: tile path
  int wd, gh, ntx, ntile;
  const int32_t* gpos; // [7][N] CSR position of SW,S,W,C,E,N,NE or -1
  int order;           // extrapolation order of the initial guess (<= kRingS - 1)
  // graph-driven step loop: the PCG while-node's condition, cleared by the
  // iteration in which the last live task of the step stops
  cudaGraphConditionalHandle it_cond;
  int use_cond;
  // region-linear operator (mlmcp_ctx_set_region_grid + per-sample region
  // parameters): the tile kernels compute the operator coefficients from the
  // six triangles around each point instead of streaming them (rcls null:
  // the stored [S][4][N] symmetric halves of A and M)
  const uint8_t* rcls;     // [N] point class (Ctx::rcls)
  const uint32_t* rckey;   // [rC] class key: six 4-bit triangle regions | neighbour mask << 24
  int rC;
  const double* rpar;      // [S][R][2] (sigma_r masked, nu_r)
  int R;
  double rmw[12], rkw[12]; // C0..C5, E0, E1, N0, N1, NE0, NE1
  Work w;
};

// Block reduce of NV values to thread 0, then the last-arriving block of the
// task reduces all partials in fixed order.  Returns true in the last block
// (all threads), with totals in v.
template <int NV>
__device__ __forceinline__ bool task_reduce(double (&v)[NV], const SArgs& a, int t,
                                            double* red, int nb = -1, int slot = -1) {
  __shared__ bool last;
  int par = 0;
  if (nb < 0) nb = a.nblk;
  if (slot < 0) slot = blockIdx.x;
  block_allsum<NV>(v, red, par);
  if (threadIdx.x == 0) {
    double* dst = a.w.partial + ((int64_t)t * a.nblk + slot) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) dst[k] = v[k];
    __threadfence();
    const int prev = atomicAdd(a.w.arrive + t, 1);
    last = (prev == nb - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const double* src = a.w.partial + ((int64_t)t * a.nblk + b) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += __ldcg(src + k);
  }
  block_allsum<NV>(acc, red, par);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = acc[k];
  if (threadIdx.x == 0) a.w.arrive[t] = 0;
  return true;
}

__device__ __forceinline__ bool task_live(const SArgs& a, const mlmcp_task& tk, int t) {
  if (a.w.ti[t * kTI + I_CODE] != MLMCP_ST_OK) return false;
  if (a.active != nullptr && tk.group >= 0 && a.active[tk.group] == 0) return false;
  return true;
}

// Block-uniform read of a flag another block may be writing: thread 0 reads,
// the block agrees (barriers below must not diverge).
__device__ __forceinline__ bool block_uniform(bool v) {
  __shared__ int flag;
  if (threadIdx.x == 0) flag = v ? 1 : 0;
  __syncthreads();
  const bool out = flag != 0;
  __syncthreads();
  return out;
}


// Last block of a task's PCG iteration (spmv / tile kernels): stopping rule
// r.D^-1.r <= rtol^2 b.D^-1.b, failure codes, and the Chronopoulos-Gear
// scalars alpha, beta of the update that follows.
__device__ __forceinline__ void cg_scalars(const SArgs& a, int t, double gamma, double delta) {
  double* td = a.w.td + t * kTD;
  int32_t* ti = a.w.ti + t * kTI;
  int code = MLMCP_ST_OK;
  bool stop = false;
  if (gamma <= a.rtol2 * td[D_BB]) {
    stop = true;
  } else if (!isfinite(gamma)) {
    code = MLMCP_ST_NONFINITE;
  } else if (ti[I_IT_STEP] >= a.max_it) {
    code = MLMCP_ST_NOCONV;
  } else if (ti[I_IT_STEP] == 0) {
    if (!(delta > 0.0)) code = MLMCP_ST_BREAKDOWN;
    else {
      td[D_ALPHA] = gamma / delta;
      td[D_BETA] = 0.0;
      td[D_GAMMA] = gamma;
    }
  } else {
    const double beta = gamma / td[D_GAMMA];
    const double den = delta - beta * gamma / td[D_ALPHA];
    if (!(den > 0.0)) code = MLMCP_ST_BREAKDOWN;
    else {
      td[D_ALPHA] = gamma / den;
      td[D_BETA] = beta;
      td[D_GAMMA] = gamma;
    }
  }
  if (code != MLMCP_ST_OK) {
    ti[I_CODE] = code;
    stop = true;
  }
  if (stop) {
    ti[I_STATE] = ST_DONE;
    const int done = atomicAdd(a.w.counters + 1, 1) + 1;
    if (a.use_cond && done >= *(volatile const int32_t*)(a.w.counters + 0))
      cudaGraphSetConditional(a.it_cond, 0);
  } else {
    ti[I_FIRST] = (ti[I_IT_STEP] == 0);
    ti[I_IT_STEP] += 1;
    ti[I_IT_TOTAL] += 1;
  }
}

__global__ void form_ell_kernel(SArgs a, double dt) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  double* As = a.w.A + (int64_t)s * a.W * a.N;
  double diag = 1.0;
  for (int j = 0; j < a.W; ++j) {
    const int q = a.ell_pos[j * a.N + i];
    double v = 0.0;
    if (q >= 0) {
      v = op_entry(Ms[q], Ks[q], dt);
      if (a.col[q] == i) diag = v;
    }
    As[(int64_t)j * a.N + i] = v;
  }
  a.w.dinv[(int64_t)s * a.N + i] = 1.0 / diag;
}

__global__ void copy_in_kernel(SArgs a) {
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.N) {
    const double x = a.xbuf[tk.x_in + i];
    a.w.X[(int64_t)t * a.N + i] = x;
    a.w.Wv[(int64_t)t * a.N + i] = x;   // a_0 for the tile path's step start
    if (tk.traj >= 0) a.xbuf[tk.traj + i] = x;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < kTI; ++k) a.w.ti[t * kTI + k] = 0;
    for (int k = 0; k < kTD; ++k) a.w.td[t * kTD + k] = 0.0;
    a.w.arrive[t] = 0;
  }
}

// Initial guess of the step (as the SM-resident path): with a periodic steady
// state X (task.ss_slot >= 0) the guess is ss_{n+1} + the order-3
// extrapolation of the transients y = a - ss; without, the order-4
// extrapolation of the states; a_n itself for MLMCP_TASK_NO_EXTRAPOLATION
// (the reference's one-step semantics).  The ring keeps y (= a when ss = 0),
// a_n moves to Wv (the rhs reads it there), X becomes the guess.
__global__ void __launch_bounds__(kThreads) guess_kernel(SArgs a, int step_arg) {
  const int step = step_arg >= 0 ? step_arg : *(volatile const int32_t*)(a.w.counters + 2);
  __shared__ double sc[4];
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const bool pred = a.xss != nullptr && tk.ss_slot >= 0 &&
                    !(tk.flags & MLMCP_TASK_NO_EXTRAPOLATION);
  if (threadIdx.x == 0 && pred) {
    const int64_t g = tk.k0 + step + 1;
    sincos(__dmul_rn(a.omega, grid_time(tk.t_base, g, tk.dt)), &sc[0], &sc[1]);
    sincos(__dmul_rn(a.omega, grid_time(tk.t_base, g - 1, tk.dt)), &sc[2], &sc[3]);
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N || step >= tk.n_steps) return;
  const int64_t TN = (int64_t)a.T * a.N, o = (int64_t)t * a.N + i;
  const double an = a.w.X[o];
  double sst = 0.0, ssn = 0.0;
  if (pred) {
    const double* Xs = a.xss + (int64_t)tk.ss_slot * 2 * a.N;
    const double xr = Xs[i], xi = Xs[a.N + i];
    sst = fma(xr, sc[0], xi * sc[1]);
    ssn = fma(xr, sc[2], xi * sc[3]);
  }
  const double yn = an - ssn;
  const int p = (tk.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : min(step, a.order);
  auto past = [&](int k) { return a.w.ring[(int64_t)((step - k) & (kRingS - 1)) * TN + o]; };
  // polynomial extrapolation of order p through y_n .. y_{n-p} (high orders pay:
  // the states are smooth in time)
  double g = yn;
  if (pred && p >= 7 && c_ls_on) {
    g = c_ls68[0] * yn;
    for (int j = 1; j < 8; ++j) g = fma(c_ls68[j], past(j), g);
  } else if (p > 0) {
    g = c_extrap[p][0] * yn;
    for (int j = 1; j <= p; ++j) g = fma(c_extrap[p][j], past(j), g);
  }
  a.w.ring[(int64_t)(step & (kRingS - 1)) * TN + o] = yn;
  a.w.Wv[o] = an;
  a.w.X[o] = g + sst;
}

// Last block of a task's step start: b.D^-1.b of the stopping rule, state
// bb = b.D^-1.b of the step; bstop (>= bb) the reference of the stopping rule
// (bb itself except for correction solves, MLMCP_TASK_CORRECTION)
__device__ __forceinline__ void step_scalars(const SArgs& a, int t, double bb, double bstop = -1.0) {
  double* td = a.w.td + t * kTD;
  int32_t* ti = a.w.ti + t * kTI;
  td[D_BB] = bstop >= 0.0 ? bstop : bb;
  ti[I_IT_STEP] = 0;
  ti[I_FIRST] = 1;
  atomicAdd(a.w.counters + 0, 1);
  if (bb == 0.0) {
    ti[I_STATE] = ST_ZERO;
    atomicAdd(a.w.counters + 1, 1);
  } else {
    ti[I_STATE] = ST_RUN;
  }
}

// rhs b = M a_n + dt*sf*prof, r = b - A x0, partial b.D^-1.b (Jacobi-weighted
// norm of the stopping rule, as the SM-resident path)
__global__ void __launch_bounds__(kThreads) step_init_kernel(SArgs a, int step_arg) {
  const int step = step_arg >= 0 ? step_arg : *(volatile const int32_t*)(a.w.counters + 2);
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  if (!block_uniform(step < tk.n_steps && task_live(a, tk, t))) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = tk.sample;
  const int64_t g = tk.k0 + step + 1;
  const double sf = sin(__dmul_rn(a.omega, grid_time(tk.t_base, g, tk.dt)));
  double bb = 0.0;
  if (i < a.N) {
    const double* X = a.w.X + (int64_t)t * a.N;
    const double* An = a.w.Wv + (int64_t)t * a.N;      // a_n (guess_kernel)
    const double* Ms = a.M + (int64_t)s * a.nnz;
    const double* As = a.w.A + (int64_t)s * a.W * a.N;
    double mx = 0.0;
    const int q0 = a.row_ptr[i], q1 = a.row_ptr[i + 1];
    for (int q = q0; q < q1; ++q) mx = fma(Ms[q], An[a.col[q]], mx);
    double ax = 0.0;
    if (a.tile) {   // A = M + dt K from the CSR values (w.A holds the tile layout)
      const double* Ks = a.K + (int64_t)s * a.nnz;
      for (int q = q0; q < q1; ++q) ax = fma(op_entry(Ms[q], Ks[q], tk.dt), X[a.col[q]], ax);
    } else {
      for (int j = 0; j < a.W; ++j)
        ax = fma(As[(int64_t)j * a.N + i], X[a.ell_col[j * a.N + i]], ax);
    }
    const double b = __dadd_rn(mx, __dmul_rn(tk.dt, __dmul_rn(sf, a.profile[i])));
    a.w.R[(int64_t)t * a.N + i] = b - ax;
    bb = b * a.w.dinv[(int64_t)s * a.N + i] * b;
  }
  double v[1] = {bb};
  if (task_reduce<1>(v, a, t, red) && threadIdx.x == 0) step_scalars(a, t, v[0]);
}

__global__ void __launch_bounds__(kThreads) spmv_kernel(SArgs a) {
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  if (!block_uniform(a.w.ti[t * kTI + I_STATE] == ST_RUN && task_live(a, tk, t))) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = tk.sample;
  double ru = 0.0, wu = 0.0, rr = 0.0;
  if (i < a.N) {
    const double* R = a.w.R + (int64_t)t * a.N;
    const double* Di = a.w.dinv + (int64_t)s * a.N;
    const double* As = a.w.A + (int64_t)s * a.W * a.N;
    double w = 0.0;
    for (int j = 0; j < a.W; ++j) {
      const int c = a.ell_col[j * a.N + i];
      w = fma(As[(int64_t)j * a.N + i], Di[c] * R[c], w);
    }
    const double r = R[i];
    const double u = Di[i] * r;
    a.w.Wv[(int64_t)t * a.N + i] = w;
    ru = r * u;
    wu = w * u;
    rr = r * r;
  }
  double v[3] = {ru, wu, rr};
  if (task_reduce<3>(v, a, t, red) && threadIdx.x == 0) cg_scalars(a, t, v[0], v[1]);
}

__global__ void __launch_bounds__(kThreads) update_kernel(SArgs a) {
  const int t = blockIdx.y;
  const int state = a.w.ti[t * kTI + I_STATE];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const int64_t o = (int64_t)t * a.N + i;
  if (state == ST_ZERO) {
    a.w.X[o] = 0.0;
    return;
  }
  if (state != ST_RUN) return;
  const mlmcp_task tk = a.tasks[t];
  const double* td = a.w.td + t * kTD;
  const double alpha = td[D_ALPHA], beta = td[D_BETA];
  const bool first = a.w.ti[t * kTI + I_FIRST] != 0;
  const double r = a.w.R[o];
  const double u = a.w.dinv[(int64_t)tk.sample * a.N + i] * r;
  const double w = a.w.Wv[o];
  const double p = first ? u : fma(beta, a.w.P[o], u);
  const double s = first ? w : fma(beta, a.w.Sv[o], w);
  a.w.P[o] = p;
  a.w.Sv[o] = s;
  a.w.X[o] = fma(alpha, p, a.w.X[o]);
  a.w.R[o] = fma(-alpha, s, r);
}

// ------------------------------------------------------------------ tile path
// Structured wd x gh grids too large for one cluster (256^2, 512^2: configs
// 2, 4): ONE launch per PCG iteration over all live (task, tile) pairs.  A
// tile is kTW x kTH grid points; each thread a column strip of kTR rows.
// Launch k (k = PCG iterations done in this step) fuses the update of
// iteration k-1 with the operator apply of iteration k:
//   p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s   (own points)
//   u = D^-1 r on the tile and its one-point halo (halo values recomputed
//   from the previous iterates of the neighbouring tiles), w = A u from the
//   shared-memory u, partial (r.u, w.u); the last tile of the task computes
//   the scalars (cg_scalars).
// r, w, s alternate between two buffers by iteration parity, so a launch reads
// only buffers no tile of the same launch writes.  The operator is the
// symmetric half (C, E, N, NE) per point, [S][4][N]; W, S, SW are the E, N, NE
// coefficients of the west / south / south-west neighbour.
// HBM streams per point and iteration: read x r w s p + 4 operator values,
// write x r w s p = 112 B (D^-1 = 1/C recomputed; B_it = 8 nnz + 56 N also
// counts 112 B).
constexpr int kTW = 64;
constexpr int kTLD = kTW + 2;

__global__ void form_tile_kernel(SArgs a, double dt) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  double* As = a.w.A + (int64_t)s * 4 * a.N;
  double* Ms4 = a.w.A + ((int64_t)a.S + s) * 4 * a.N;   // mass, same layout
  double c = 1.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int q = a.gpos[(int64_t)(3 + j) * a.N + i];
    const double v = q >= 0 ? op_entry(Ms[q], Ks[q], dt) : 0.0;
    if (j == 0 && q >= 0) c = v;
    As[(int64_t)j * a.N + i] = v;
    Ms4[(int64_t)j * a.N + i] = q >= 0 ? Ms[q] : 0.0;
  }
  a.w.dinv[(int64_t)s * a.N + i] = 1.0 / c;
}

// Region-linear operator of one point class (Ctx::rckey): the six triangles
// around the point (code: their regions, 4 bits each, in increasing element
// order e0..e5 = SWl, SWu, Su, Wl, Ol, Ou), which of the SW, S, W, E, N, NE
// neighbours are interior points (mask bits 0..5), and the task's region
// parameters sp[r] = (sigma_r, nu_r).  Every stencil coefficient of the point
// couples it to a neighbour through triangles that touch the point, so all
// seven are available here: C over e0..e5, E over (e2, e4), N (e3, e5),
// NE (e4, e5), and W (e1, e3), S (e0, e2), SW (e0, e1) — the E, N, NE of the
// west, south and south-west neighbours with the same weights, hence the same
// doubles.  Sums run in the assembly gather map's element order with
// assemble_kernel's and op_entry's arithmetic: bitwise the CSR values
// mlmcp_assemble writes.  Slot order SW, S, W, C, E, N, NE (the CSR column
// order of a row).
__device__ __forceinline__ void region_stencil(const SArgs& a, const double2* sp, uint32_t code,
                                               uint32_t mask, double dt, double (&A)[7],
                                               double (&Mo)[7]) {
  double2 p[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) p[e] = sp[(code >> (4 * e)) & 15u];
  double m = 0.0, k = 0.0;
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    m = __dadd_rn(m, __dmul_rn(p[e].x, a.rmw[e]));
    k = __dadd_rn(k, __dmul_rn(p[e].y, a.rkw[e]));
  }
  Mo[3] = m;
  A[3] = op_entry(m, k, dt);
  //                      SW      S       W       E       N       NE
  const int slot[6] = {0, 1, 2, 4, 5, 6};
  const int e0[6] = {0, 0, 1, 2, 3, 4}, e1[6] = {1, 2, 3, 4, 5, 5};
  const int cw[6] = {10, 8, 6, 6, 8, 10};
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const bool ok = (mask >> c) & 1u;
    double mm = 0.0, kk = 0.0;
    if (ok) {
      mm = __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[c]].x, a.rmw[cw[c]])),
                     __dmul_rn(p[e1[c]].x, a.rmw[cw[c] + 1]));
      kk = __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[c]].y, a.rkw[cw[c]])),
                     __dmul_rn(p[e1[c]].y, a.rkw[cw[c] + 1]));
    }
    Mo[slot[c]] = mm;
    A[slot[c]] = ok ? op_entry(mm, kk, dt) : 0.0;
  }
}

// The task's stencils, one per point class (once per propagate call; every
// tile launch of the task copies them into shared memory, load_class_table):
// tab[d * rC + c] holds A's slot d (0..6), tab[7 * rC + c] = 1 / A_C (the
// Jacobi weight), tab[(8 + d) * rC + c] the mass matrix's slot d.
__device__ __forceinline__ void load_region_params(const SArgs& a, int sample, double2* sp);
__global__ void class_table_kernel(SArgs a) {
  __shared__ double2 sp[16];
  const int t = blockIdx.x;
  const mlmcp_task tk = a.tasks[t];
  load_region_params(a, tk.sample, sp);
  __syncthreads();
  const int C = a.rC;
  double* tab = a.w.ctab + (int64_t)t * 15 * C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const uint32_t key = __ldg(a.rckey + c);
    double A7[7], M7[7];
    region_stencil(a, sp, key & 0x00ffffffu, key >> 24, tk.dt, A7, M7);
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      tab[d * C + c] = A7[d];
      tab[(8 + d) * C + c] = M7[d];
    }
    tab[7 * C + c] = 1.0 / A7[3];
  }
}

// the first `rows` rows of task t's class table into shared memory (caller syncs)
__device__ __forceinline__ void load_class_table(const SArgs& a, int t, double* tab, int rows) {
  const int n = rows * a.rC;
  const double* g = a.w.ctab + (int64_t)t * 15 * a.rC;
  for (int i = threadIdx.x; i < n; i += blockDim.x) tab[i] = __ldg(g + i);
}

// the task's region parameters into shared memory (block-wide; caller syncs)
__device__ __forceinline__ void load_region_params(const SArgs& a, int sample, double2* sp) {
  if (threadIdx.x < a.R)
    sp[threadIdx.x] = reinterpret_cast<const double2*>(a.rpar)[(int64_t)sample * a.R + threadIdx.x];
}

__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ int bcast_int(int v) {
  __shared__ int val;
  if (threadIdx.x == 0) val = v;
  __syncthreads();
  const int out = val;
  __syncthreads();
  return out;
}

// r_k of a point from the previous iterates (identical arithmetic for the
// owner and for the neighbours that recompute it as halo)
__device__ __forceinline__ double tile_s(bool first, double beta, double wo, double so) {
  return first ? wo : fma(beta, so, wo);
}

template <int kTH, int kTR, int kMinB>
__global__ void __launch_bounds__(kTW * (kTH / kTR), kMinB) tile_iter_kernel(SArgs a) {
  constexpr int kTHalo = 2 * (kTW + 2) + 2 * kTH;
  constexpr int kNT = kTW * (kTH / kTR);
  constexpr int kTCL = kTW + 1;                 // operator tile: columns -1..kTW-1
  constexpr int kTCN = (kTH + 1) * kTCL;        //                rows -1..kTH-1
  extern __shared__ __align__(16) double tsm[];
  double* U = tsm;                              // (kTH + 2) * kTLD
  double* Ac = U + (kTH + 2) * kTLD;            // C, E, N, NE (cp.async-staged)
  __shared__ double red[2 * 4 * 32];
  // programmatic dependent launch: this grid may be scheduled while the
  // previous iteration's grid drains; wait for it (and its memory) before
  // reading anything, and let the next iteration's grid be scheduled early
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const int32_t* ti = a.w.ti + t * kTI;
  int mode = 0;   // 0 skip, 1 run, 2 zero solution
  if (threadIdx.x == 0 && task_live(a, tk, t)) {
    const int st = ti[I_STATE];
    mode = st == ST_RUN ? 1 : (st == ST_ZERO ? 2 : 0);
  }
  mode = bcast_int(mode);
  if (mode == 0) return;
  const int k = ti[I_IT_STEP];
  const int64_t N = a.N, o = (int64_t)t * N;
  const int tx0 = (blockIdx.x % a.ntx) * kTW, ty0 = (blockIdx.x / a.ntx) * kTH;
  const int cx = threadIdx.x % kTW, sy = threadIdx.x / kTW;
  const int gx = tx0 + cx;
  const int gy0 = ty0 + sy * kTR;
  const bool colok = gx < a.wd;
  double* X = a.w.X + o;
  if (mode == 2) {
#pragma unroll
    for (int r = 0; r < kTR; ++r)
      if (colok && gy0 + r < a.gh) X[(int64_t)(gy0 + r) * a.wd + gx] = 0.0;
    return;
  }
  const double* Di = a.w.dinv + (int64_t)tk.sample * N;
  const double* As = a.w.A + (int64_t)tk.sample * 4 * N;
  // operator of the tile and of its west column / south row: asynchronous
  // copies into shared memory, overlapped with the vector loads below
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int ly = sy * kTR + r;
    const bool ok = colok && gy0 + r < a.gh;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) cp8(&Ac[j * kTCN + (ly + 1) * kTCL + cx + 1], As + j * N + i, ok);
  }
  for (int h = threadIdx.x; h < kTH + 1 + kTW; h += kNT) {
    const int lx = h <= kTH ? -1 : h - (kTH + 1), ly = h <= kTH ? h - 1 : -1;
    const int hx = tx0 + lx, hy = ty0 + ly;
    const bool ok = hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh;
    const int64_t j = ok ? (int64_t)hy * a.wd + hx : 0;
#pragma unroll
    for (int q = 1; q < 4; ++q) cp8(&Ac[q * kTCN + (ly + 1) * kTCL + lx + 1], As + q * N + j, ok);
  }
  cp_commit();
  const bool odd = k & 1, upd = k > 0, first = k == 1;
  const double* td = a.w.td + t * kTD;
  const double alpha = upd ? td[D_ALPHA] : 0.0, beta = upd ? td[D_BETA] : 0.0;
  // parity buffers: r_j in R[j&1], w_j in W[j&1], s_j in S[j&1] (buffer 0 = R, Wv, Sv)
  const double* Ro = (odd || !upd) ? a.w.R + o : a.w.R1 + o;   // r_{k-1} (k == 0: r_0)
  const double* Wo = odd ? a.w.Wv + o : a.w.W1 + o;            // w_{k-1}
  const double* So = odd ? a.w.S1 + o : a.w.Sv + o;            // s_{k-2}
  double* Rn = odd ? a.w.R1 + o : a.w.R + o;
  double* Sn = odd ? a.w.Sv + o : a.w.S1 + o;
  double* Wn = odd ? a.w.W1 + o : a.w.Wv + o;

  // halo frame: u at the neighbouring tiles' points (0 outside the grid)
  for (int h = threadIdx.x; h < kTHalo; h += kNT) {
    int lx, ly;
    if (h < kTW + 2) { lx = h - 1; ly = -1; }
    else if (h < 2 * (kTW + 2)) { lx = h - (kTW + 2) - 1; ly = kTH; }
    else if (h < 2 * (kTW + 2) + kTH) { lx = -1; ly = h - 2 * (kTW + 2); }
    else { lx = kTW; ly = h - 2 * (kTW + 2) - kTH; }
    const int hx = tx0 + lx, hy = ty0 + ly;
    double u = 0.0;
    if (hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh) {
      const int64_t j = (int64_t)hy * a.wd + hx;
      double r = __ldcg(Ro + j);
      if (upd) r = fma(-alpha, tile_s(first, beta, __ldcg(Wo + j), first ? 0.0 : __ldcg(So + j)), r);
      u = __ldg(Di + j) * r;
    }
    U[(ly + 1) * kTLD + lx + 1] = u;
  }
  // own points: update of iteration k-1, u_k
  double gam = 0.0;
  {
    double rv[kTR], dv[kTR], wv[kTR], sv[kTR], pv[kTR], xv[kTR];
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
      rv[r] = ok ? __ldcg(Ro + i) : 0.0;
      if (upd) {
        wv[r] = ok ? __ldcg(Wo + i) : 0.0;
        sv[r] = (ok && !first) ? __ldcg(So + i) : 0.0;
        pv[r] = (ok && !first) ? __ldcg(a.w.P + o + i) : 0.0;
        xv[r] = ok ? __ldcg(X + i) : 0.0;
      }
    }
    // D^-1 of the own points from the staged diagonal (this thread's own
    // copies: no barrier needed), the same correctly rounded 1/C as
    // form_tile_kernel's stored D^-1 (one 8-byte stream less per iteration)
    cp_wait_all();
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      dv[r] = ok ? 1.0 / Ac[(sy * kTR + r + 1) * kTCL + cx + 1] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
      double rk = rv[r];
      if (upd) {
        const double uo = dv[r] * rv[r];
        const double p = first ? uo : fma(beta, pv[r], uo);
        const double s = tile_s(first, beta, wv[r], sv[r]);
        rk = fma(-alpha, s, rv[r]);
        if (ok) {
          a.w.P[o + i] = p;
          Sn[i] = s;
          X[i] = fma(alpha, p, xv[r]);
          Rn[i] = rk;
        }
      }
      const double u = dv[r] * rk;
      U[(sy * kTR + r + 1) * kTLD + cx + 1] = u;
      gam = fma(rk, u, gam);
    }
  }
  cp_wait_all();
  __syncthreads();
  // w_k = A u_k (W, S, SW coefficients = E, N, NE of the west / south / south-west point)
  double del = 0.0;
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int gy = gy0 + r;
    if (!(colok && gy < a.gh)) continue;
    const int64_t i = (int64_t)gy * a.wd + gx;
    const int b = (sy * kTR + r + 1) * kTLD + cx + 1;
    const int lc = (sy * kTR + r + 1) * kTCL + cx + 1;
    const double c = Ac[lc], e = Ac[kTCN + lc], nn = Ac[2 * kTCN + lc], ne = Ac[3 * kTCN + lc];
    const double cw = Ac[kTCN + lc - 1];
    const double cs = Ac[2 * kTCN + lc - kTCL];
    const double csw = Ac[3 * kTCN + lc - kTCL - 1];
    const double uc = U[b];
    double acc0 = c * uc, acc1 = csw * U[b - kTLD - 1];
    acc0 = fma(cs, U[b - kTLD], acc0);
    acc1 = fma(cw, U[b - 1], acc1);
    acc0 = fma(e, U[b + 1], acc0);
    acc1 = fma(nn, U[b + kTLD], acc1);
    acc0 = fma(ne, U[b + kTLD + 1], acc0);
    const double w = acc0 + acc1;
    Wn[i] = w;
    del = fma(w, uc, del);
  }
  double v[2] = {gam, del};
  if (task_reduce<2>(v, a, t, red, a.ntile) && threadIdx.x == 0) cg_scalars(a, t, v[0], v[1]);
}

// Region-mode iteration kernel (mlmcp_ctx_set_region_grid): tile_iter_kernel's
// arithmetic with the operator computed from the task's region parameters
// instead of streamed.  Every global load of the launch (task state, own-point
// vectors, the thread's halo point, the point classes) is issued before any
// dependent arithmetic; while they are in flight the CTA forms the task's
// stencil of every point class (build_class_table: a few dozen classes, one
// per thread), and each point then reads its seven coefficients and its
// Jacobi weight from that table.  Shared memory: u with its halo (9.5 KB) and
// the table (8 doubles per class).  HBM per point: read x r w s p, write
// x r w s p = 80 B (the 1-byte point classes are shared by every task and stay
// in L2).
template <int kTH, int kTR, int kMinB>
__global__ void __launch_bounds__(kTW * (kTH / kTR), kMinB) tile_iter_rg_kernel(SArgs a) {
  constexpr int kTHalo = 2 * (kTW + 2) + 2 * kTH;
  constexpr int kNT = kTW * (kTH / kTR);
  static_assert(kTHalo <= kNT, "one halo point per thread");
  extern __shared__ __align__(16) double tsm[];
  double* U = tsm;                              // (kTH + 2) * kTLD
  double* tab = tsm + (kTH + 2) * kTLD;         // [8][rC] class stencils, 1 / A_C
  __shared__ double red[2 * 4 * 32];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  // task state: every thread reads it (same addresses: broadcast loads; the
  // previous launch has completed, and this launch's last tile of task t
  // writes it only after every tile of t has read it)
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const int32_t* ti = a.w.ti + t * kTI;
  const double* td = a.w.td + t * kTD;
  const int st = ti[I_STATE];
  const int k = ti[I_IT_STEP];
  const int code_ok = ti[I_CODE];
  const int act = (a.active != nullptr && tk.group >= 0) ? a.active[tk.group] : 1;
  const double alpha_l = td[D_ALPHA], beta_l = td[D_BETA];
  if (code_ok != MLMCP_ST_OK || act == 0 || (st != ST_RUN && st != ST_ZERO)) return;
  const int64_t N = a.N, o = (int64_t)t * N;
  const int tx0 = (blockIdx.x % a.ntx) * kTW, ty0 = (blockIdx.x / a.ntx) * kTH;
  const int cx = threadIdx.x % kTW, sy = threadIdx.x / kTW;
  const int gx = tx0 + cx;
  const int gy0 = ty0 + sy * kTR;
  const bool colok = gx < a.wd;
  double* X = a.w.X + o;
  if (st == ST_ZERO) {
#pragma unroll
    for (int r = 0; r < kTR; ++r)
      if (colok && gy0 + r < a.gh) X[(int64_t)(gy0 + r) * a.wd + gx] = 0.0;
    return;
  }
  const bool odd = k & 1, upd = k > 0, first = k == 1;
  const double alpha = upd ? alpha_l : 0.0, beta = upd ? beta_l : 0.0;
  const double* Ro = (odd || !upd) ? a.w.R + o : a.w.R1 + o;   // r_{k-1} (k == 0: r_0)
  const double* Wo = odd ? a.w.Wv + o : a.w.W1 + o;            // w_{k-1}
  const double* So = odd ? a.w.S1 + o : a.w.Sv + o;            // s_{k-2}
  double* Rn = odd ? a.w.R1 + o : a.w.R + o;
  double* Sn = odd ? a.w.Sv + o : a.w.S1 + o;
  double* Wn = odd ? a.w.W1 + o : a.w.Wv + o;
  // ---- 1. every global load of the launch, issued up front
  double rv[kTR], wv[kTR], sv[kTR], pv[kTR], xv[kTR];
  int cd[kTR];
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const bool ok = colok && gy0 + r < a.gh;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
    cd[r] = ok ? (int)__ldg(a.rcls + i) : 0;
    rv[r] = ok ? __ldcg(Ro + i) : 0.0;
    wv[r] = (ok && upd) ? __ldcg(Wo + i) : 0.0;
    sv[r] = (ok && upd && !first) ? __ldcg(So + i) : 0.0;
    pv[r] = (ok && upd && !first) ? __ldcg(a.w.P + o + i) : 0.0;
    xv[r] = (ok && upd) ? __ldcg(X + i) : 0.0;
  }
  int hb = -1;                 // shared-memory slot of this thread's halo point
  double hr = 0.0, hw = 0.0, hs = 0.0;
  int hcl = -1;                // halo point's class (-1: outside the grid)
  if (threadIdx.x < kTHalo) {
    const int h = threadIdx.x;
    int lx, ly;
    if (h < kTW + 2) { lx = h - 1; ly = -1; }
    else if (h < 2 * (kTW + 2)) { lx = h - (kTW + 2) - 1; ly = kTH; }
    else if (h < 2 * (kTW + 2) + kTH) { lx = -1; ly = h - 2 * (kTW + 2); }
    else { lx = kTW; ly = h - 2 * (kTW + 2) - kTH; }
    hb = (ly + 1) * kTLD + lx + 1;
    const int hx = tx0 + lx, hy = ty0 + ly;
    if (hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh) {
      const int64_t j = (int64_t)hy * a.wd + hx;
      hcl = (int)__ldg(a.rcls + j);
      hr = __ldcg(Ro + j);
      if (upd) {
        hw = __ldcg(Wo + j);
        if (!first) hs = __ldcg(So + j);
      }
    }
  }
  load_class_table(a, t, tab, 8);
  __syncthreads();
  const int C = a.rC;
  // ---- 2. the halo point: u = D^-1 r_k with D = C of that point
  if (hb >= 0) {
    double u = 0.0;
    if (hcl >= 0) {
      double r = hr;
      if (upd) r = fma(-alpha, tile_s(first, beta, hw, hs), r);
      u = tab[7 * C + hcl] * r;
    }
    U[hb] = u;
  }
  // ---- 3. own points: update of iteration k-1, u_k
  double gam = 0.0;
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const bool ok = colok && gy0 + r < a.gh;
    const double dv = ok ? tab[7 * C + cd[r]] : 0.0;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
    double rk = rv[r];
    if (upd) {
      const double uo = dv * rv[r];
      const double p = first ? uo : fma(beta, pv[r], uo);
      const double sn = tile_s(first, beta, wv[r], sv[r]);
      rk = fma(-alpha, sn, rv[r]);
      if (ok) {
        a.w.P[o + i] = p;
        Sn[i] = sn;
        X[i] = fma(alpha, p, xv[r]);
        Rn[i] = rk;
      }
    }
    const double u = dv * rk;
    U[(sy * kTR + r + 1) * kTLD + cx + 1] = u;
    gam = fma(rk, u, gam);
  }
  __syncthreads();
  // ---- 4. w_k = A u_k with the point's own stencil, partial (r.u, w.u)
  double del = 0.0;
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int gy = gy0 + r;
    if (!(colok && gy < a.gh)) continue;
    const int64_t i = (int64_t)gy * a.wd + gx;
    const int b = (sy * kTR + r + 1) * kTLD + cx + 1;
    double A7[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) A7[d] = tab[d * C + cd[r]];
    const double uc = U[b];
    double acc0 = A7[3] * uc, acc1 = A7[0] * U[b - kTLD - 1];
    acc0 = fma(A7[1], U[b - kTLD], acc0);
    acc1 = fma(A7[2], U[b - 1], acc1);
    acc0 = fma(A7[4], U[b + 1], acc0);
    acc1 = fma(A7[5], U[b + kTLD], acc1);
    acc0 = fma(A7[6], U[b + kTLD + 1], acc0);
    const double w = acc0 + acc1;
    Wn[i] = w;
    del = fma(w, uc, del);
  }
  double v[2] = {gam, del};
  if (task_reduce<2>(v, a, t, red, a.ntile) && threadIdx.x == 0) cg_scalars(a, t, v[0], v[1]);
}

// 7-point stencil product at smem offset b (row stride ld), in the summation
// order of tile_iter_kernel: every path forms w = A u with the same doubles.
template <int ld>
__device__ __forceinline__ double stencil_apply(const double* U, int b, const double (&A7)[7]) {
  double acc0 = A7[3] * U[b], acc1 = A7[0] * U[b - ld - 1];
  acc0 = fma(A7[1], U[b - ld], acc0);
  acc1 = fma(A7[2], U[b - 1], acc1);
  acc0 = fma(A7[4], U[b + 1], acc0);
  acc1 = fma(A7[5], U[b + ld], acc1);
  acc0 = fma(A7[6], U[b + ld + 1], acc0);
  return acc0 + acc1;
}

// Region-mode iteration kernel without a stored w (the default in region
// mode): launch k recomputes w_{k-1} = A u_{k-1} from r_{k-1} instead of
// reading it, so a PCG iteration streams read r s p x, write r s p x = 64 B
// per point (tile_iter_rg_kernel: 80 B).  Launch k:
//   u_{k-1} = D^-1 r_{k-1} on the tile + a two-point halo (r_{k-1} read there),
//   w_{k-1} = A u_{k-1}, s_{k-1} = w_{k-1} + beta s_{k-2}, r_k = r_{k-1} - alpha
//   s_{k-1}, u_k = D^-1 r_k on the tile + the one-point halo,
//   p_{k-1} = u_{k-1} + beta p_{k-2}, x_k = x_{k-1} + alpha p_{k-1} (own points),
//   w_k = A u_k (own points), partials (r_k.u_k, w_k.u_k);
// launch 0 only forms u_0, w_0 and the partials.  Every value is computed with
// tile_iter_kernel's arithmetic (stencil_apply, tile_s), so the iterates are
// bitwise those of the stored-w kernels.  r and s keep their parity buffers
// (a launch never writes what a neighbouring tile reads); p and x are
// own-point only and updated in place.
template <int kTH, int kTR, int kMinB>
__global__ void __launch_bounds__(kTW * (kTH / kTR), kMinB) tile_iter_rw_kernel(SArgs a) {
  constexpr int kNT = kTW * (kTH / kTR);
  constexpr int kL1 = kTW + 4;                      // smem row stride (two-point frame)
  constexpr int kR1 = 2 * (kTW + 2) + 2 * kTH;      // one-point ring (164 at 64 x 16)
  constexpr int kR2 = 2 * (kTW + 4) + 2 * (kTH + 2);  // second ring (172)
  static_assert(kR1 <= kNT && kR2 <= kNT, "one ring point per thread and ring");
  extern __shared__ __align__(16) double tsm[];
  double* U1 = tsm;                                 // u_{k-1}: (kTH + 4) x kL1
  double* U2 = tsm + (kTH + 4) * kL1;               // u_k, same frame
  double* tab = U2 + (kTH + 4) * kL1;               // [8][rC]
  __shared__ double red[2 * 4 * 32];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const int32_t* ti = a.w.ti + t * kTI;
  const double* td = a.w.td + t * kTD;
  const int st = ti[I_STATE];
  const int k = ti[I_IT_STEP];
  const int code_ok = ti[I_CODE];
  const int act = (a.active != nullptr && tk.group >= 0) ? a.active[tk.group] : 1;
  const double alpha_l = td[D_ALPHA], beta_l = td[D_BETA];
  if (code_ok != MLMCP_ST_OK || act == 0 || (st != ST_RUN && st != ST_ZERO)) return;
  const int64_t N = a.N, o = (int64_t)t * N;
  const int tx0 = (blockIdx.x % a.ntx) * kTW, ty0 = (blockIdx.x / a.ntx) * kTH;
  const int cx = threadIdx.x % kTW, sy = threadIdx.x / kTW;
  const int gx = tx0 + cx;
  const int gy0 = ty0 + sy * kTR;
  const bool colok = gx < a.wd;
  double* X = a.w.X + o;
  if (st == ST_ZERO) {
#pragma unroll
    for (int r = 0; r < kTR; ++r)
      if (colok && gy0 + r < a.gh) X[(int64_t)(gy0 + r) * a.wd + gx] = 0.0;
    return;
  }
  const bool odd = k & 1, upd = k > 0, first = k == 1;
  const double alpha = upd ? alpha_l : 0.0, beta = upd ? beta_l : 0.0;
  const double* Ro = (odd || !upd) ? a.w.R + o : a.w.R1 + o;   // r_{k-1} (k == 0: r_0)
  const double* So = odd ? a.w.S1 + o : a.w.Sv + o;            // s_{k-2}
  double* Rn = odd ? a.w.R1 + o : a.w.R + o;
  double* Sn = odd ? a.w.Sv + o : a.w.S1 + o;
  // ---- 1. every global load, issued up front
  double rv[kTR], sv[kTR], pv[kTR], xv[kTR];
  int cd[kTR];
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const bool ok = colok && gy0 + r < a.gh;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
    cd[r] = ok ? (int)__ldg(a.rcls + i) : 0;
    rv[r] = ok ? __ldcg(Ro + i) : 0.0;
    sv[r] = (ok && upd && !first) ? __ldcg(So + i) : 0.0;
    pv[r] = (ok && upd && !first) ? __ldcg(a.w.P + o + i) : 0.0;
    xv[r] = (ok && upd) ? __ldcg(X + i) : 0.0;
  }
  // one-point ring point of this thread (threads < kR1): r_{k-1}, s_{k-2}, class
  int b1 = -1, c1 = -1;            // smem offset; class (-1: outside the grid)
  double r1 = 0.0, s1 = 0.0;
  if (threadIdx.x < kR1) {
    const int h = threadIdx.x;
    int lx, ly;
    if (h < kTW + 2) { lx = h - 1; ly = -1; }
    else if (h < 2 * (kTW + 2)) { lx = h - (kTW + 2) - 1; ly = kTH; }
    else if (h < 2 * (kTW + 2) + kTH) { lx = -1; ly = h - 2 * (kTW + 2); }
    else { lx = kTW; ly = h - 2 * (kTW + 2) - kTH; }
    b1 = (ly + 2) * kL1 + lx + 2;
    const int hx = tx0 + lx, hy = ty0 + ly;
    if (hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh) {
      const int64_t j = (int64_t)hy * a.wd + hx;
      c1 = (int)__ldg(a.rcls + j);
      r1 = __ldcg(Ro + j);
      if (upd && !first) s1 = __ldcg(So + j);
    }
  }
  // second ring point (threads >= kNT - kR2, launches k >= 1): r_{k-1}, class
  int b2 = -1, c2 = -1;
  double r2 = 0.0;
  if (upd && threadIdx.x >= kNT - kR2) {
    const int h = threadIdx.x - (kNT - kR2);
    int lx, ly;
    if (h < kTW + 4) { lx = h - 2; ly = -2; }
    else if (h < 2 * (kTW + 4)) { lx = h - (kTW + 4) - 2; ly = kTH + 1; }
    else if (h < 2 * (kTW + 4) + kTH + 2) { lx = -2; ly = h - 2 * (kTW + 4) - 1; }
    else { lx = kTW + 1; ly = h - 2 * (kTW + 4) - (kTH + 2) - 1; }
    b2 = (ly + 2) * kL1 + lx + 2;
    const int hx = tx0 + lx, hy = ty0 + ly;
    if (hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh) {
      const int64_t j = (int64_t)hy * a.wd + hx;
      c2 = (int)__ldg(a.rcls + j);
      r2 = __ldcg(Ro + j);
    }
  }
  load_class_table(a, t, tab, 8);
  __syncthreads();
  const int C = a.rC;
  const double* Dv = tab + 7 * C;
#ifdef MLMCP_CHECKED
  for (int r = 0; r < kTR; ++r) MLMCP_DCHECK(cd[r] >= 0 && cd[r] < C);
  MLMCP_DCHECK(c1 < C && c2 < C);
  MLMCP_DCHECK(b1 < (kTH + 4) * kL1 && b2 < (kTH + 4) * kL1);
  MLMCP_DCHECK((int64_t)(gy0 + kTR - 1) * a.wd + gx < N || !colok || gy0 + kTR - 1 >= a.gh);
#endif
  double gam = 0.0;
  if (upd) {
    // ---- 2. u_{k-1} on the tile and the two-point frame
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      U1[(sy * kTR + r + 2) * kL1 + cx + 2] = ok ? Dv[cd[r]] * rv[r] : 0.0;
    }
    if (b1 >= 0) U1[b1] = c1 >= 0 ? Dv[c1] * r1 : 0.0;
    if (b2 >= 0) U1[b2] = c2 >= 0 ? Dv[c2] * r2 : 0.0;
    __syncthreads();
    // ---- 3. w_{k-1}, s_{k-1}, r_k, u_k on the tile and the one-point ring
    if (b1 >= 0) {
      double u = 0.0;
      if (c1 >= 0) {
        double A7[7];
#pragma unroll
        for (int d = 0; d < 7; ++d) A7[d] = tab[d * C + c1];
        const double w = stencil_apply<kL1>(U1, b1, A7);
        const double rk = fma(-alpha, tile_s(first, beta, w, s1), r1);
        u = Dv[c1] * rk;
      }
      U2[b1] = u;
    }
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      const int b = (sy * kTR + r + 2) * kL1 + cx + 2;
      double u = 0.0;
      if (ok) {
        const int64_t i = (int64_t)(gy0 + r) * a.wd + gx;
        double A7[7];
#pragma unroll
        for (int d = 0; d < 7; ++d) A7[d] = tab[d * C + cd[r]];
        const double w = stencil_apply<kL1>(U1, b, A7);
        const double uo = U1[b];
        const double p = first ? uo : fma(beta, pv[r], uo);
        const double sn = tile_s(first, beta, w, sv[r]);
        const double rk = fma(-alpha, sn, rv[r]);
        a.w.P[o + i] = p;
        Sn[i] = sn;
        X[i] = fma(alpha, p, xv[r]);
        Rn[i] = rk;
        u = Dv[cd[r]] * rk;
        gam = fma(rk, u, gam);
      }
      U2[b] = u;
    }
  } else {
    // ---- launch 0: u_0 on the tile and the one-point ring
    if (b1 >= 0) U2[b1] = c1 >= 0 ? Dv[c1] * r1 : 0.0;
#pragma unroll
    for (int r = 0; r < kTR; ++r) {
      const bool ok = colok && gy0 + r < a.gh;
      const double u = ok ? Dv[cd[r]] * rv[r] : 0.0;
      U2[(sy * kTR + r + 2) * kL1 + cx + 2] = u;
      gam = fma(rv[r], u, gam);
    }
  }
  __syncthreads();
  // ---- 4. w_k = A u_k on the own points, partial (r.u, w.u)
  double del = 0.0;
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    if (!(colok && gy0 + r < a.gh)) continue;
    const int b = (sy * kTR + r + 2) * kL1 + cx + 2;
    double A7[7];
#pragma unroll
    for (int d = 0; d < 7; ++d) A7[d] = tab[d * C + cd[r]];
    const double w = stencil_apply<kL1>(U2, b, A7);
    del = fma(w, U2[b], del);
  }
  double v[2] = {gam, del};
  if (task_reduce<2>(v, a, t, red, a.ntile) && threadIdx.x == 0) cg_scalars(a, t, v[0], v[1]);
}

template <int kTH, int kTR>
constexpr size_t tile_iter_rw_smem(int n_classes = 256) {
  return sizeof(double) * (2 * (kTH + 4) * (kTW + 4) + 8 * n_classes);
}

template <int kTH, int kTR>
constexpr size_t tile_iter_rg_smem(int n_classes = 256) {
  return sizeof(double) * ((kTH + 2) * kTLD + 8 * n_classes);
}

template <int kTH, int kTR>
constexpr size_t tile_iter_smem() {
  return sizeof(double) * ((kTH + 2) * kTLD + 4 * (kTH + 1) * (kTW + 1));
}

// MLMCP_TILE_RW=0: region mode keeps the stored-w iteration kernel (A/B)
bool rw_on() {
  const char* e = getenv("MLMCP_TILE_RW");
  return !(e && atoi(e) == 0);
}

// launch one tile iteration (programmatic dependent launch unless disabled)
template <int kTH, int kTR, int kMinB>
int launch_tile_iter(const SArgs& a, dim3 grid, cudaStream_t s, bool pdl) {
  constexpr int nt = kTW * (kTH / kTR);
  constexpr size_t smem = tile_iter_smem<kTH, kTR>();
  static bool attr = false;
  if (!attr) {
    MLMCP_CUDA_CHECK(cudaFuncSetAttribute(tile_iter_kernel<kTH, kTR, kMinB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MLMCP_CUDA_CHECK(cudaFuncSetAttribute(tile_iter_rg_kernel<kTH, kTR, kMinB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)tile_iter_rg_smem<kTH, kTR>()));
    MLMCP_CUDA_CHECK(cudaFuncSetAttribute(tile_iter_rw_kernel<kTH, kTR, kMinB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)tile_iter_rw_smem<kTH, kTR>()));
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = dim3(nt);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  if (a.rcls != nullptr && rw_on()) {
    lc.dynamicSmemBytes = tile_iter_rw_smem<kTH, kTR>(a.rC);
    MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&lc, tile_iter_rw_kernel<kTH, kTR, kMinB>, a));
    MLMCP_LAUNCH_CHECK("tile_iter_rw_kernel");
  } else if (a.rcls != nullptr) {
    lc.dynamicSmemBytes = tile_iter_rg_smem<kTH, kTR>(a.rC);
    MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&lc, tile_iter_rg_kernel<kTH, kTR, kMinB>, a));
    MLMCP_LAUNCH_CHECK("tile_iter_rg_kernel");
  } else {
    MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&lc, tile_iter_kernel<kTH, kTR, kMinB>, a));
    MLMCP_LAUNCH_CHECK("tile_iter_kernel");
  }
  return MLMCP_OK;
}

// Step start on the tile layout: b = M a_n + dt sf profile, r_0 = b - A x_0,
// partial b.D^-1.b.  a_n (Wv) and x_0 (X) are staged with their one-point
// halo, the symmetric halves of A and M with their west column / south row,
// all by cp.async; the stencil sums run in the CSR column order
// (SW, S, W, C, E, N, NE) of the per-row kernel.
template <int kTH, int kTR, int kMinB>
__global__ void __launch_bounds__(kTW * (kTH / kTR), kMinB) tile_init_kernel(SArgs a, int step_arg) {
  const int step = step_arg >= 0 ? step_arg : *(volatile const int32_t*)(a.w.counters + 2);
  constexpr int kTCL = kTW + 1, kTCN = (kTH + 1) * kTCL, kTV = (kTH + 2) * kTLD;
  constexpr int kTHalo = 2 * (kTW + 2) + 2 * kTH;
  static_assert(kTHalo <= kTW * (kTH / kTR), "one halo point per thread");
  extern __shared__ __align__(16) double ism[];
  const bool region = a.rcls != nullptr;
  // region mode: the task's stencils per point class (build_class_table, A and
  // M) instead of the staged operator
  double* Ac = ism;                                  // [4][kTCN] (stored operator)
  double* XV = region ? ism : Ac + 4 * kTCN;         // x_0 with halo
  double* AV = XV + kTV;                             // a_n with halo
  double* tab = AV + kTV;                            // region: [15][rC]
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  if (!block_uniform(step < tk.n_steps && task_live(a, tk, t))) return;
  const int64_t N = a.N, o = (int64_t)t * N;
  const int tx0 = (blockIdx.x % a.ntx) * kTW, ty0 = (blockIdx.x / a.ntx) * kTH;
  const int cx = threadIdx.x % kTW, sy = threadIdx.x / kTW;
  const int gx = tx0 + cx, gy0 = ty0 + sy * kTR;
  const bool colok = gx < a.wd;
  const double* As = a.w.A + (int64_t)tk.sample * 4 * N;
  const double* Ms = a.w.A + ((int64_t)a.S + tk.sample) * 4 * N;
  const double* An = a.w.Wv + o;   // a_n (step_end / copy_in)
  double dv[kTR];
  if (region) load_class_table(a, t, tab, 15);   // visible after the guess's sync
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int ly = sy * kTR + r;
    const bool ok = colok && gy0 + r < a.gh;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
    const int lc = (ly + 1) * kTCL + cx + 1, lv = (ly + 1) * kTLD + cx + 1;
    if (!region) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cp8(&Ac[j * kTCN + lc], As + j * N + i, ok);
    }
    cp8(&AV[lv], An + i, ok);
  }
  if (!region && threadIdx.x < kTH + 1 + kTW) {
    const int h = threadIdx.x;
    const int lx = h <= kTH ? -1 : h - (kTH + 1), ly = h <= kTH ? h - 1 : -1;
    const int hx = tx0 + lx, hy = ty0 + ly;
    const bool ok = hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh;
    const int64_t j = ok ? (int64_t)hy * a.wd + hx : 0;
    const int lc = (ly + 1) * kTCL + lx + 1;
#pragma unroll
    for (int q = 1; q < 4; ++q) cp8(&Ac[q * kTCN + lc], As + q * N + j, ok);
  }
  if (threadIdx.x < kTHalo) {
    int lx, ly;
    const int h = threadIdx.x;
    if (h < kTW + 2) { lx = h - 1; ly = -1; }
    else if (h < 2 * (kTW + 2)) { lx = h - (kTW + 2) - 1; ly = kTH; }
    else if (h < 2 * (kTW + 2) + kTH) { lx = -1; ly = h - 2 * (kTW + 2); }
    else { lx = kTW; ly = h - 2 * (kTW + 2) - kTH; }
    const int hx = tx0 + lx, hy = ty0 + ly;
    const bool ok = hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh;
    const int64_t j = ok ? (int64_t)hy * a.wd + hx : 0;
    const int lv = (ly + 1) * kTLD + lx + 1;
    cp8(&AV[lv], An + j, ok);
  }
  cp_commit();
  // initial guess x_0 (the guess kernel's arithmetic, folded in) for the own
  // points and the halo frame; a_n comes from Wv (written by step_end / copy_in),
  // so no tile reads what another tile writes (X, ring slot step & 7)
  __shared__ double sc[4];
  const bool pred = a.xss != nullptr && tk.ss_slot >= 0 &&
                    !(tk.flags & MLMCP_TASK_NO_EXTRAPOLATION);
  if (threadIdx.x == 0 && pred) {
    const int64_t gg = tk.k0 + step + 1;
    sincos(__dmul_rn(a.omega, grid_time(tk.t_base, gg, tk.dt)), &sc[0], &sc[1]);
    sincos(__dmul_rn(a.omega, grid_time(tk.t_base, gg - 1, tk.dt)), &sc[2], &sc[3]);
  }
  __syncthreads();
  const int pord = (tk.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : min(step, a.order);
  const int64_t TN = (int64_t)a.T * N;
  const double* Xs = pred ? a.xss + (int64_t)tk.ss_slot * 2 * N : nullptr;
  // x_0 at task point j from a_n (an); y_n joins the ring when `own`
  auto guess_at = [&](int64_t j, double an, bool own) {
    double sst = 0.0, ssn = 0.0;
    if (pred) {
      const double xr = __ldg(Xs + j), xi = __ldg(Xs + N + j);
      sst = fma(xr, sc[0], xi * sc[1]);
      ssn = fma(xr, sc[2], xi * sc[3]);
    }
    const double yn = an - ssn;
    double pv[kRingS];   // past transients, loaded together (independent loads)
#pragma unroll
    for (int q = 1; q < kRingS; ++q)
      pv[q] = q <= pord ? __ldcg(a.w.ring + (int64_t)((step - q) & (kRingS - 1)) * TN + o + j) : 0.0;
    double gv = yn;
    if (pred && pord >= 7 && c_ls_on) {
      gv = c_ls68[0] * yn;
#pragma unroll
      for (int q = 1; q < 8; ++q) gv = fma(c_ls68[q], pv[q], gv);
    } else if (pord > 0) {
      gv = c_extrap[pord][0] * yn;
#pragma unroll
      for (int q = 1; q < kRingS; ++q)
        if (q <= pord) gv = fma(c_extrap[pord][q], pv[q], gv);
    }
    if (own) a.w.ring[(int64_t)(step & (kRingS - 1)) * TN + o + j] = yn;
    return gv + sst;
  };
  const int64_t g = tk.k0 + step + 1;
  const bool corr = (tk.flags & MLMCP_TASK_CORRECTION) != 0;
  const double sf = corr ? 0.0 : sin(__dmul_rn(a.omega, grid_time(tk.t_base, g, tk.dt)));
  double prof[kTR];
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const bool ok = colok && gy0 + r < a.gh;
    const int64_t i = ok ? (int64_t)(gy0 + r) * a.wd + gx : 0;
    prof[r] = ok ? __ldg(a.profile + i) : 0.0;
    if (!region) dv[r] = ok ? __ldg(a.w.dinv + (int64_t)tk.sample * N + i) : 0.0;
  }
  cp_wait_all();   // own and halo a_n were copied by this thread
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int ly = sy * kTR + r;
    const bool ok = colok && gy0 + r < a.gh;
    const int lv = (ly + 1) * kTLD + cx + 1;
    double x0 = 0.0;
    if (ok) {
      const int64_t i = (int64_t)(gy0 + r) * a.wd + gx;
      x0 = guess_at(i, AV[lv], true);
      a.w.X[o + i] = x0;
    }
    XV[lv] = x0;
  }
  if (threadIdx.x < kTHalo) {
    int lx, ly;
    const int h = threadIdx.x;
    if (h < kTW + 2) { lx = h - 1; ly = -1; }
    else if (h < 2 * (kTW + 2)) { lx = h - (kTW + 2) - 1; ly = kTH; }
    else if (h < 2 * (kTW + 2) + kTH) { lx = -1; ly = h - 2 * (kTW + 2); }
    else { lx = kTW; ly = h - 2 * (kTW + 2) - kTH; }
    const int hx = tx0 + lx, hy = ty0 + ly;
    const int lv = (ly + 1) * kTLD + lx + 1;
    double x0 = 0.0;
    if (hx >= 0 && hx < a.wd && hy >= 0 && hy < a.gh)
      x0 = guess_at((int64_t)hy * a.wd + hx, AV[lv], false);
    XV[lv] = x0;
  }
  __syncthreads();
  double bb = 0.0, bref = 0.0;
#pragma unroll
  for (int r = 0; r < kTR; ++r) {
    const int ly = sy * kTR + r, gy = gy0 + r;
    if (!(colok && gy < a.gh)) continue;
    const int64_t i = (int64_t)gy * a.wd + gx;
    const int lc = (ly + 1) * kTCL + cx + 1, b = (ly + 1) * kTLD + cx + 1;
    // coefficient of direction SW, S, W, C, E, N, NE (A staged; M from global:
    // own C, E, N, NE and the E, N, NE of the west / south / south-west points)
    const int cofs[7] = {3 * kTCN + lc - kTCL - 1, 2 * kTCN + lc - kTCL, kTCN + lc - 1, lc,
                         kTCN + lc, 2 * kTCN + lc, 3 * kTCN + lc};
    const int vofs[7] = {b - kTLD - 1, b - kTLD, b - 1, b, b + 1, b + kTLD, b + kTLD + 1};
    const bool w_ = gx > 0, s_ = gy > 0;
    double mco[7], aco[7];
    if (region) {
      const int C = a.rC, c = (int)__ldg(a.rcls + i);
#pragma unroll
      for (int d = 0; d < 7; ++d) {
        aco[d] = tab[d * C + c];
        mco[d] = tab[(8 + d) * C + c];
      }
      dv[r] = tab[7 * C + c];
    } else {
#pragma unroll
      for (int d = 0; d < 7; ++d) aco[d] = Ac[cofs[d]];
      mco[0] = (w_ && s_) ? __ldg(Ms + 3 * N + i - a.wd - 1) : 0.0;
      mco[1] = s_ ? __ldg(Ms + 2 * N + i - a.wd) : 0.0;
      mco[2] = w_ ? __ldg(Ms + N + i - 1) : 0.0;
      mco[3] = __ldg(Ms + i);
      mco[4] = __ldg(Ms + N + i);
      mco[5] = __ldg(Ms + 2 * N + i);
      mco[6] = __ldg(Ms + 3 * N + i);
    }
    double mx = 0.0, ax = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      mx = fma(mco[d], AV[vofs[d]], mx);
      ax = fma(aco[d], XV[vofs[d]], ax);
    }
    const double bv = __dadd_rn(mx, __dmul_rn(tk.dt, __dmul_rn(sf, prof[r])));
    a.w.R[o + i] = bv - ax;
    bb += bv * dv[r] * bv;
    if (corr) {   // reference magnitude: the diagonal part of M applied to the corrected solution
      const double mf = mco[3] * __ldcg(a.xbuf + tk.x_out + i);
      bref += mf * dv[r] * mf;
    }
  }
  if (corr) {   // block-uniform (one task per blockIdx.y)
    double v[2] = {bb, bref};
    if (task_reduce<2>(v, a, t, red, a.ntile) && threadIdx.x == 0)
      step_scalars(a, t, v[0], fmax(v[0], v[1]));
    return;
  }
  double v[1] = {bb};
  if (task_reduce<1>(v, a, t, red, a.ntile) && threadIdx.x == 0) step_scalars(a, t, v[0]);
}

template <int kTH, int kTR>
constexpr size_t tile_init_smem(bool region = false, int n_classes = 256) {
  return sizeof(double) * ((region ? 15 * n_classes : 4 * (kTH + 1) * (kTW + 1)) +
                           2 * (kTH + 2) * kTLD);
}


// mode 0: per-step (trajectory store + SUM_ENERGY accumulation);
// mode 1: finalize (x_out, FINAL_ENERGY / SUM write-out, iters, status)
__global__ void __launch_bounds__(kThreads) step_end_kernel(SArgs a, int step_arg, int mode) {
  const int step = step_arg >= 0 ? step_arg : *(volatile const int32_t*)(a.w.counters + 2);
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const mlmcp_task tk = a.tasks[t];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int32_t* ti = a.w.ti + t * kTI;
  double* td = a.w.td + t * kTD;
  const bool inactive = block_uniform(a.active != nullptr && tk.group >= 0 &&
                                      a.active[tk.group] == 0 && ti[I_CODE] == MLMCP_ST_OK);
  if (inactive) return;
  const double* X = a.w.X + (int64_t)t * a.N;
  const double* Ks = a.K + (int64_t)tk.sample * a.nnz;
  bool energy = false;
  const int code_now = block_uniform(ti[I_CODE] != MLMCP_ST_OK) ? 1 : 0;
  if (mode == 0) {
    if (step >= tk.n_steps || code_now) return;
    if (tk.traj >= 0 && i < a.N) a.xbuf[tk.traj + (int64_t)(step + 1) * a.N + i] = X[i];
    if (a.tile && i < a.N) a.w.Wv[(int64_t)t * a.N + i] = X[i];   // a_n of the next step
    const int64_t g = tk.k0 + step + 1;
    energy = tk.qoi_mode == MLMCP_QOI_SUM_ENERGY && g > tk.qoi_from && tk.qoi_slot >= 0;
  } else {
    if (tk.x_out >= 0 && i < a.N) {
      if (tk.flags & MLMCP_TASK_CORRECTION) a.xbuf[tk.x_out + i] += X[i];
      else a.xbuf[tk.x_out + i] = X[i];
    }
    energy = tk.qoi_mode == MLMCP_QOI_FINAL_ENERGY && tk.qoi_slot >= 0 && !code_now;
  }
  double e = 0.0;
  if (energy && i < a.N) {
    double kx = 0.0;
    for (int q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) kx = fma(Ks[q], X[a.col[q]], kx);
    e = X[i] * kx;
  }
  if (energy) {
    double v[1] = {e};
    if (task_reduce<1>(v, a, t, red) && threadIdx.x == 0) {
      if (mode == 0) td[D_ACC] += 0.5 * v[0];
      else a.qoi[tk.qoi_slot] = 0.5 * v[0];
    }
  }
  if (mode == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    if (tk.qoi_mode == MLMCP_QOI_SUM_ENERGY && tk.qoi_slot >= 0) a.qoi[tk.qoi_slot] = td[D_ACC];
    if (a.iters != nullptr && tk.slot >= 0) a.iters[tk.slot] = ti[I_IT_TOTAL];
    if (ti[I_CODE] != MLMCP_ST_OK) {
      write_status(a.status, tk.slot, ti[I_CODE], ti[I_FAILSTEP], tk.tag, tk.tag);
      if (a.active != nullptr && tk.group >= 0) a.active[tk.group] = 0;
    }
  }
}

// records the failing step of tasks that failed in this step
__global__ void mark_fail_kernel(SArgs a, int step_arg) {
  const int step = step_arg >= 0 ? step_arg : *(volatile const int32_t*)(a.w.counters + 2);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  int32_t* ti = a.w.ti + t * kTI;
  if (ti[I_CODE] != MLMCP_ST_OK && ti[I_FAILSTEP] < 0) ti[I_FAILSTEP] = step;
  if (ti[I_CODE] == MLMCP_ST_OK) ti[I_FAILSTEP] = -1;
}

// control kernels of the graph-driven step loop (counters[2] = current step)
__global__ void steps_begin_kernel(int32_t* counters) { counters[2] = 0; }

// PCG while-node condition at the start of a step: run while live tasks remain
__global__ void iter_begin_kernel(int32_t* counters, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, counters[1] < counters[0] ? 1 : 0);
}

__global__ void step_next_kernel(int32_t* counters, int n_steps, cudaGraphConditionalHandle h) {
  const int s = counters[2] + 1;
  counters[2] = s;
  cudaGraphSetConditional(h, s < n_steps ? 1 : 0);
}

// extrapolation order of the streaming paths' initial guesses (MLMCP_STREAM_ORDER)
// MLMCP_LSGUESS=0: exact extrapolation instead of the least-squares guess
int ls_on() {
  const char* l = getenv("MLMCP_LSGUESS");
  return (l && atoi(l) == 0) ? 0 : 1;
}

int stream_order() {
  const char* e = getenv("MLMCP_STREAM_ORDER");
  const int o = e ? atoi(e) : 7;   // measured: cfg2 10.0 -> 6.3, cfg4 8.6 -> 6.7 its/step vs order 4
  return std::max(0, std::min(o, kRingS - 1));
}

// MLMCP_STREAM_IMPL: 1 two-launch ELL kernels, 2 cooperative, 3 cluster,
// 4 tile; default auto
int stream_impl() {
  const char* e = getenv("MLMCP_STREAM_IMPL");
  return e ? atoi(e) : 0;
}

bool tile_usable(const Ctx* ctx) {
  const int impl = stream_impl();
  if (impl == 1 || impl == 2) return false;
  if (ctx->cl_wd == 0 || ctx->n < kTW) return false;
  const int ntile = ((ctx->cl_wd + 63) / 64) * ((ctx->cl_h + 15) / 16);   // finest tiling
  return ntile <= (ctx->n + kThreads - 1) / kThreads;   // partial-sum slots
}

// MLMCP_TILE_CFG: 1 default (<16,4,3>; the recompute-w region kernel <16,4,4>),
// 2 <16,4,4>, 3 <8,2,4>; 64x32 tiles at 2 CTAs/SM measured 11% slower than the
// default.  (A warp-specialised variant staging tiles with cp.async.bulk row
// copies measured 2.3x slower and was removed.)
int tile_cfg() {
  const char* e = getenv("MLMCP_TILE_CFG");
  return e ? std::max(1, std::min(3, atoi(e))) : 1;
}

// MLMCP_TILE_PDL=0 disables programmatic dependent launch of the tile
// iterations (back-to-back launches then drain fully before the next starts)
bool pdl_on() {
  const char* e = getenv("MLMCP_TILE_PDL");
  return !(e && atoi(e) == 0);
}

// MLMCP_STREAM_GRAPH=1: device-driven step loop (conditional graph nodes);
// measured on par with the host loop below (whose syncs overlap nothing
// costly), which stays the default because ncu can profile its kernels
bool graph_steps() {
  const char* e = getenv("MLMCP_STREAM_GRAPH");
  return e && atoi(e) == 1;
}

// three private non-blocking streams for building the step graph by capture
int capture_streams(Ctx* ctx, cudaStream_t (&cs)[3]) {
  for (int i = 0; i < 3; ++i) {
    if (ctx->cap_stream[i] == nullptr) {
      cudaError_t e = cudaStreamCreateWithFlags(&ctx->cap_stream[i], cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreateWithFlags");
    }
    cs[i] = ctx->cap_stream[i];
  }
  return MLMCP_OK;
}

// instantiate (or update the cached executable graph in place) and launch
int launch_exec(Ctx* ctx, cudaGraph_t g, cudaStream_t stream) {
  if (ctx->step_exec != nullptr) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ctx->step_exec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(ctx->step_exec);
      ctx->step_exec = nullptr;
    }
  }
  if (ctx->step_exec == nullptr) {
    cudaError_t e = cudaGraphInstantiate(&ctx->step_exec, g, 0);
    if (e != cudaSuccess) {
      ctx->step_exec = nullptr;
      return cuda_fail(e, "cudaGraphInstantiate(step loop)");
    }
  }
  MLMCP_CUDA_CHECK(cudaGraphLaunch(ctx->step_exec, stream));
  return MLMCP_OK;
}

int run_steps(Ctx* ctx, SArgs& a, int n_steps_max, double dt, cudaStream_t stream) {
  const dim3 blk(kThreads);
  const dim3 grid_rows((a.N + kThreads - 1) / kThreads, a.T);
  const dim3 grid_form((a.N + kThreads - 1) / kThreads, a.S);
  if (a.tile) {
    if (a.rcls == nullptr) {   // region mode computes the operator in the tile kernels
      form_tile_kernel<<<grid_form, blk, 0, stream>>>(a, dt);
      MLMCP_LAUNCH_CHECK("form_tile_kernel");
    }
  } else {
    form_ell_kernel<<<grid_form, blk, 0, stream>>>(a, dt);
    MLMCP_LAUNCH_CHECK("form_ell_kernel");
  }
  const int tcfg = tile_cfg();
  if (a.tile) {   // 64-column tiles of 16 rows (variants 3, 4: 8 rows)
    const int th = tcfg >= 3 ? 8 : 16;
    a.ntx = (a.wd + kTW - 1) / kTW;
    a.ntile = a.ntx * ((a.gh + th - 1) / th);
  }
  const dim3 grid_tiles2(a.tile ? a.ntile : 1, a.T);
  copy_in_kernel<<<grid_rows, blk, 0, stream>>>(a);
  MLMCP_LAUNCH_CHECK("copy_in_kernel");
  if (a.rcls != nullptr) {
    class_table_kernel<<<a.T, 64, 0, stream>>>(a);
    MLMCP_LAUNCH_CHECK("class_table_kernel");
  }
  mark_fail_kernel<<<(a.T + 255) / 256, 256, 0, stream>>>(a, 0);
  MLMCP_LAUNCH_CHECK("mark_fail_kernel");
  auto launch_init = [&](cudaStream_t s, int step) -> int {
    const bool rg = a.rcls != nullptr;
    if (a.tile && tcfg >= 3) {
      tile_init_kernel<8, 2, 4><<<grid_tiles2, 256, tile_init_smem<8, 2>(rg, a.rC), s>>>(a, step);
      MLMCP_LAUNCH_CHECK("tile_init_kernel");
    } else if (a.tile) {
      tile_init_kernel<16, 4, 3><<<grid_tiles2, 256, tile_init_smem<16, 4>(rg, a.rC), s>>>(a, step);
      MLMCP_LAUNCH_CHECK("tile_init_kernel");
    } else {
      step_init_kernel<<<grid_rows, blk, 0, s>>>(a, step);
      MLMCP_LAUNCH_CHECK("step_init_kernel");
    }
    return MLMCP_OK;
  };
  if (a.tile) {
    static bool attr = false;
    if (!attr) {
      MLMCP_CUDA_CHECK(cudaFuncSetAttribute(tile_init_kernel<8, 2, 4>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)std::max(tile_init_smem<8, 2>(false),
                                                          tile_init_smem<8, 2>(true))));
      MLMCP_CUDA_CHECK(cudaFuncSetAttribute(tile_init_kernel<16, 4, 3>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)std::max(tile_init_smem<16, 4>(false),
                                                          tile_init_smem<16, 4>(true))));
      attr = true;
    }
  }
  auto launch_iteration = [&](cudaStream_t s) -> int {
    if (a.tile) {
      if (tcfg == 1 && !(a.rcls != nullptr && rw_on())) {
        if (const int rc = launch_tile_iter<16, 4, 3>(a, grid_tiles2, s, pdl_on())) return rc;
      } else if (tcfg == 1) {
        // the recompute-w kernel fits 64 registers: 4 CTAs per SM (config 4:
        // 154 -> 140 ms on the iteration launches, scripts/tile_ab.py region@2)
        if (const int rc = launch_tile_iter<16, 4, 4>(a, grid_tiles2, s, pdl_on())) return rc;
      } else if (tcfg == 2) {
        if (const int rc = launch_tile_iter<16, 4, 4>(a, grid_tiles2, s, pdl_on())) return rc;
      } else {
        if (const int rc = launch_tile_iter<8, 2, 4>(a, grid_tiles2, s, pdl_on())) return rc;
      }
    } else {
      spmv_kernel<<<grid_rows, blk, 0, s>>>(a);
      MLMCP_LAUNCH_CHECK("spmv_kernel");
      update_kernel<<<grid_rows, blk, 0, s>>>(a);
      MLMCP_LAUNCH_CHECK("update_kernel");
    }
    return MLMCP_OK;
  };
  if (graph_steps()) {
    // Device-driven step loop: one CUDA graph with a while-node over the steps
    // whose body runs the step's kernels and a nested while-node over PCG
    // iterations; the iteration in which the last task stops clears the inner
    // condition (cg_scalars).  No host synchronisation per step or iteration.
    if (n_steps_max <= 0) {
      step_end_kernel<<<grid_rows, blk, 0, stream>>>(a, 0, 1);
      MLMCP_LAUNCH_CHECK("step_end_kernel(final)");
      return MLMCP_OK;
    }
    cudaStream_t cs[3];
    if (const int rc0 = capture_streams(ctx, cs)) return rc0;
    cudaGraph_t g;
    MLMCP_CUDA_CHECK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_step, h_it;
    MLMCP_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h_step, g, 1, cudaGraphCondAssignDefault));
    // the step loop (body graph b_step)
    cudaGraphNodeParams ps = {};
    ps.type = cudaGraphNodeTypeConditional;
    ps.conditional.handle = h_step;
    ps.conditional.type = cudaGraphCondTypeWhile;
    ps.conditional.size = 1;
    cudaGraphNode_t n_step;
    MLMCP_CUDA_CHECK(cudaGraphAddNode(&n_step, g, nullptr, 0, &ps));
    cudaGraph_t b_step = ps.conditional.phGraph_out[0];
    MLMCP_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h_it, b_step, 0, 0));
    a.it_cond = h_it;
    a.use_cond = 1;
    // body of the step loop: guess, rhs, the PCG loop, step end, advance
    MLMCP_CUDA_CHECK(cudaStreamBeginCaptureToGraph(cs[1], b_step, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal));
    int rc = MLMCP_OK;
    do {
      if (cudaMemsetAsync(a.w.counters, 0, 2 * sizeof(int32_t), cs[1]) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "cudaMemsetAsync");
        break;
      }
      if (!a.tile) guess_kernel<<<grid_rows, blk, 0, cs[1]>>>(a, -1);
      rc = launch_init(cs[1], -1);
      if (rc != MLMCP_OK) break;
      iter_begin_kernel<<<1, 1, 0, cs[1]>>>(a.w.counters, h_it);
      cudaStreamCaptureStatus st;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      cudaGraph_t cap;
      if (cudaStreamGetCaptureInfo(cs[1], &st, nullptr, &cap, &deps, &nd) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "cudaStreamGetCaptureInfo");
        break;
      }
      cudaGraphNodeParams pi = {};
      pi.type = cudaGraphNodeTypeConditional;
      pi.conditional.handle = h_it;
      pi.conditional.type = cudaGraphCondTypeWhile;
      pi.conditional.size = 1;
      cudaGraphNode_t n_it;
      if (cudaGraphAddNode(&n_it, cap, deps, nd, &pi) != cudaSuccess ||
          cudaStreamUpdateCaptureDependencies(cs[1], &n_it, 1,
                                              cudaStreamSetCaptureDependencies) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "conditional node");
        break;
      }
      cudaGraph_t b_it = pi.conditional.phGraph_out[0];
      if (cudaStreamBeginCaptureToGraph(cs[2], b_it, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "capture (iteration body)");
        break;
      }
      rc = launch_iteration(cs[2]);
      cudaGraph_t b_it_out;
      const cudaError_t e2 = cudaStreamEndCapture(cs[2], &b_it_out);
      if (rc == MLMCP_OK && e2 != cudaSuccess) rc = cuda_fail(e2, "end capture (iteration body)");
      if (rc != MLMCP_OK) break;
      mark_fail_kernel<<<(a.T + 255) / 256, 256, 0, cs[1]>>>(a, -1);
      step_end_kernel<<<grid_rows, blk, 0, cs[1]>>>(a, -1, 0);
      step_next_kernel<<<1, 1, 0, cs[1]>>>(a.w.counters, n_steps_max, h_step);
    } while (false);
    cudaGraph_t b_step_out;
    const cudaError_t e1 = cudaStreamEndCapture(cs[1], &b_step_out);
    if (rc == MLMCP_OK && e1 != cudaSuccess) rc = cuda_fail(e1, "end capture (step body)");
    if (rc == MLMCP_OK) {
      steps_begin_kernel<<<1, 1, 0, stream>>>(a.w.counters);
      rc = launch_exec(ctx, g, stream);
    }
    cudaGraphDestroy(g);
    if (rc != MLMCP_OK) return rc;
    MLMCP_LAUNCH_CHECK("graph step loop");
    step_end_kernel<<<grid_rows, blk, 0, stream>>>(a, 0, 1);
    MLMCP_LAUNCH_CHECK("step_end_kernel(final)");
    return MLMCP_OK;
  }
  int32_t* hc = ctx->host_counters;
  int chunk = 4;
  for (int step = 0; step < n_steps_max; ++step) {
    MLMCP_CUDA_CHECK(cudaMemsetAsync(a.w.counters, 0, 2 * sizeof(int32_t), stream));
    if (!a.tile) {   // the tile path's step start computes the guess itself
      guess_kernel<<<grid_rows, blk, 0, stream>>>(a, step);
      MLMCP_LAUNCH_CHECK("guess_kernel");
    }
    if (const int rc = launch_init(stream, step)) return rc;
    int done_iters = 0;
    for (;;) {
      if (ctx->time_iters) MLMCP_CUDA_CHECK(cudaEventRecord(ctx->iter_ev[0], stream));
      for (int c = 0; c < chunk; ++c) {
        const int rc = launch_iteration(stream);
        if (rc != MLMCP_OK) return rc;
      }
      if (ctx->time_iters) MLMCP_CUDA_CHECK(cudaEventRecord(ctx->iter_ev[1], stream));
      done_iters += chunk;
      MLMCP_CUDA_CHECK(cudaMemcpyAsync(hc, a.w.counters, 2 * sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, stream));
      MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
      if (ctx->time_iters) {
        float ms = 0.0f;
        MLMCP_CUDA_CHECK(cudaEventElapsedTime(&ms, ctx->iter_ev[0], ctx->iter_ev[1]));
        ctx->iter_ms += ms;
        ctx->iter_launches += chunk;
      }
      if (hc[1] >= hc[0]) break;
      chunk = 2;
    }
    chunk = std::max(2, done_iters - 1);
    mark_fail_kernel<<<(a.T + 255) / 256, 256, 0, stream>>>(a, step);
    MLMCP_LAUNCH_CHECK("mark_fail_kernel");
    step_end_kernel<<<grid_rows, blk, 0, stream>>>(a, step, 0);
    MLMCP_LAUNCH_CHECK("step_end_kernel");
  }
  step_end_kernel<<<grid_rows, blk, 0, stream>>>(a, 0, 1);
  MLMCP_LAUNCH_CHECK("step_end_kernel(final)");
  return MLMCP_OK;
}

SArgs make_args(Ctx* ctx, int T, int S, const mlmcp_task* tasks, const double* M,
                const double* K, const double* profile, double omega, double rtol, int max_it,
                double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                const int32_t* active, const Work& w) {
  SArgs a;
  a.T = T;
  a.S = S;
  a.N = ctx->n;
  a.W = ctx->max_row_nnz;
  a.nblk = (ctx->n + kThreads - 1) / kThreads;
  a.nnz = ctx->nnz;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.ell_col = ctx->ell_col;
  a.ell_pos = ctx->ell_pos;
  a.tasks = tasks;
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
  a.xss = nullptr;
  a.tile = tile_usable(ctx) ? 1 : 0;
  a.wd = ctx->cl_wd;
  a.gh = ctx->cl_h;
  a.ntx = a.tile ? (a.wd + kTW - 1) / kTW : 0;
  a.ntile = a.tile ? a.ntx * ((a.gh + 15) / 16) : 0;   // set per kernel in run_steps
  a.gpos = ctx->cl_pos;
  a.it_cond = 0;
  a.use_cond = 0;
  a.order = stream_order();
  a.rcls = nullptr;
  a.rckey = nullptr;
  a.rC = 0;
  a.rpar = nullptr;
  a.R = 0;
  for (int i = 0; i < 12; ++i) a.rmw[i] = a.rkw[i] = 0.0;
  static bool ls_set = false;
  if (!ls_set) {
    const char* l = getenv("MLMCP_LSGUESS");
    if (l) {
      const int v = atoi(l) != 0;
      cudaMemcpyToSymbol(c_ls_on, &v, sizeof(int));
    }
    ls_set = true;
  }
  a.w = w;
  return a;
}

// MLMCP_TILE_OPERATOR=stored keeps the streamed [S][4][N] operator (A/B)
bool region_on() {
  const char* e = getenv("MLMCP_TILE_OPERATOR");
  return !(e && e[0] == 's');
}

// region-linear operator on the tile path when the context has a region grid
// and the caller passed the per-sample region parameters (the TMA variant
// keeps the streamed operator)
void set_region(const Ctx* ctx, SArgs& a, const double* rpar) {
  if (!a.tile || ctx->rcls == nullptr || rpar == nullptr || !region_on())
    return;
  a.rcls = ctx->rcls;
  a.rckey = ctx->rckey;
  a.rC = ctx->rC;
  a.rpar = rpar;
  a.R = ctx->rR;
  for (int i = 0; i < 12; ++i) {
    a.rmw[i] = ctx->rmw[i];
    a.rkw[i] = ctx->rkw[i];
  }
}

// Parareal correction for the streaming path: (parareal.py:168-178)
//   k == 1: U[n] = C[n-1] = c;   k >= 2: U[n] = (F[n] + c) - C[n-1]; C[n-1] = c
__global__ void correct_kernel(int S, int m, int N, int n, int k, const double* cval,
                               double* U, const double* F, double* C, const int32_t* active,
                               const int32_t* status) {
  const int s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double c = cval[(int64_t)s * N + i];
  double* Us = U + (int64_t)s * (m + 1) * N;
  const double* Fs = F + (int64_t)s * (m + 1) * N;
  double* Cs = C + (int64_t)s * m * N;
  if (k == 1) {
    Us[(int64_t)n * N + i] = c;
    Cs[(int64_t)(n - 1) * N + i] = c;
  } else {
    Us[(int64_t)n * N + i] = (Fs[(int64_t)n * N + i] + c) - Cs[(int64_t)(n - 1) * N + i];
    Cs[(int64_t)(n - 1) * N + i] = c;
  }
}

__global__ void freeze_kernel(int S, int m, int N, int idx_dst, int idx_src, double* U,
                              const double* F, const int32_t* active) {
  const int s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  U[((int64_t)s * (m + 1) + idx_dst) * N + i] = F[((int64_t)s * (m + 1) + idx_src) * N + i];
}

__global__ void coarse_status_kernel(int S, int k, int n, const int32_t* tstatus,
                                     int32_t* status, int32_t* active) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int32_t* ts = tstatus + (int64_t)s * kStatusInts;
  if (ts[0] != MLMCP_ST_OK && status[(int64_t)s * kStatusInts] == MLMCP_ST_OK) {
    write_status(status, s, ts[0], ts[1], n, k);
    active[s] = 0;
  }
}


// ---------------------------------------------------------------- steady states
// Periodic steady state X of the implicit-Euler iteration for meshes that do
// not fit one SM (the streaming counterpart of small_periodic_kernel):
// (Zr + i Zi) X = dt profile with Zr = (1 - cos w dt) M + dt K, Zi = sin(w dt) M,
// by COCG with the complex Jacobi preconditioner, one (sample, dt) item per
// blockIdx.y, the operator applied from the CSR values on the fly.  Per item
// workspace: x, r, p, z, q (complex) and D^-1 (complex) = 12 N doubles.
struct PArgs {
  int T, N, nblk;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const int32_t* sample;
  const double* dt;
  const double* M;
  const double* K;
  const double* profile;
  double omega, rtol2;
  int max_it;
  double* vec;       // [T][12][N]
  double* partial;   // [T][nblk][4]
  double* td;        // [T][8]: rho_r, rho_i, bb, alpha_r, alpha_i, beta_r, beta_i, -
  int32_t* ti;       // [T][4]: state, iters
  int32_t* arrive;   // [T]
  int32_t* counters; // [0] live, [1] done
  double* X;         // [T][2][N] output
  // region-linear operator (structured grid with a region grid + per-sample
  // region parameters): Z = (1 - e^{-i w dt}) M + dt K from the task's stencil
  // of each point class instead of the streamed CSR values of M and K
  const uint8_t* rcls;
  const uint32_t* rckey;
  int rC, R, wd;
  const double* rpar;
  double rmw[12], rkw[12];
  double* ctab;      // [T][rC][16]: Re Z (7), Re D^-1, Im Z (7), Im D^-1
};

enum : int { PV_XR = 0, PV_XI, PV_RR, PV_RI, PV_PR, PV_PI, PV_ZR, PV_ZI, PV_QR, PV_QI, PV_DR,
             PV_DI, kPV };

__device__ __forceinline__ double* pvec(const PArgs& a, int t, int k) {
  return a.vec + ((int64_t)t * kPV + k) * a.N;
}

template <int NV>
__device__ __forceinline__ bool ptask_reduce(double (&v)[NV], const PArgs& a, int t, double* red) {
  __shared__ bool last;
  int par = 0;
  block_allsum<NV>(v, red, par);
  if (threadIdx.x == 0) {
    double* dst = a.partial + ((int64_t)t * a.nblk + blockIdx.x) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) dst[k] = v[k];
    __threadfence();
    last = atomicAdd(a.arrive + t, 1) == a.nblk - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < a.nblk; b += blockDim.x) {
    const double* src = a.partial + ((int64_t)t * a.nblk + b) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += __ldcg(src + k);
  }
  block_allsum<NV>(acc, red, par);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = acc[k];
  if (threadIdx.x == 0) a.arrive[t] = 0;
  return true;
}

__device__ __forceinline__ void item_cs(const PArgs& a, int t, double& c1, double& sn,
                                        double& dt) {
  dt = a.dt[t];
  double c;
  sincos(__dmul_rn(a.omega, dt), &sn, &c);
  c1 = 1.0 - c;
}

__global__ void __launch_bounds__(kThreads) pinit_kernel(PArgs a) {
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double c1, sn, dt;
  item_cs(a, t, c1, sn, dt);
  double v[3] = {0.0, 0.0, 0.0};
  if (i < a.N) {
    const int s = a.sample[t];
    const double* Ms = a.M + (int64_t)s * a.nnz;
    const double* Ks = a.K + (int64_t)s * a.nnz;
    double m = 0.0, k = 0.0;
    for (int q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q)
      if (a.col[q] == i) {
        m = Ms[q];
        k = Ks[q];
      }
    const double dr = fma(c1, m, dt * k), di = sn * m, den = dr * dr + di * di;
    const double ir = den > 0.0 ? dr / den : 0.0, ii = den > 0.0 ? -di / den : 0.0;
    const double b = dt * a.profile[i];
    pvec(a, t, PV_DR)[i] = ir;
    pvec(a, t, PV_DI)[i] = ii;
    pvec(a, t, PV_XR)[i] = 0.0;
    pvec(a, t, PV_XI)[i] = 0.0;
    pvec(a, t, PV_RR)[i] = b;
    pvec(a, t, PV_RI)[i] = 0.0;
    pvec(a, t, PV_PR)[i] = ir * b;     // p = z = D^-1 r (r real)
    pvec(a, t, PV_PI)[i] = ii * b;
    v[0] = b * ir * b;                 // rho = r^T z (unconjugated)
    v[1] = b * ii * b;
    v[2] = b * b;
  }
  if (ptask_reduce<3>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.td + t * 8;
    td[0] = v[0];
    td[1] = v[1];
    td[2] = v[2];
    a.ti[t * 4 + 0] = v[2] > 0.0 ? 1 : 0;
    a.ti[t * 4 + 1] = 0;
    atomicAdd(a.counters + 0, 1);
    if (!(v[2] > 0.0)) atomicAdd(a.counters + 1, 1);
  }
}

// q = Z p, sigma = p^T q; last block: alpha = rho / sigma
__global__ void __launch_bounds__(kThreads) pspmv_kernel(PArgs a) {
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  if (!block_uniform(a.ti[t * 4] == 1)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double c1, sn, dt;
  item_cs(a, t, c1, sn, dt);
  double v[2] = {0.0, 0.0};
  if (i < a.N) {
    const int s = a.sample[t];
    const double* Ms = a.M + (int64_t)s * a.nnz;
    const double* Ks = a.K + (int64_t)s * a.nnz;
    const double* pr = pvec(a, t, PV_PR);
    const double* pi = pvec(a, t, PV_PI);
    double mr = 0.0, mi = 0.0, kr = 0.0, ki = 0.0;
    for (int q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) {
      const int c = a.col[q];
      const double xr = pr[c], xi = pi[c];
      const double mq = __ldcs(Ms + q), kq = __ldcs(Ks + q);   // read once: evict first
      mr = fma(mq, xr, mr);
      mi = fma(mq, xi, mi);
      kr = fma(kq, xr, kr);
      ki = fma(kq, xi, ki);
    }
    // Zr p = c1 M p + dt K p;  Zi p = sn M p;  q = Zr p + i Zi p
    const double zr_r = fma(c1, mr, dt * kr), zr_i = fma(c1, mi, dt * ki);
    const double qr = zr_r - sn * mi, qi = zr_i + sn * mr;
    __stcs(pvec(a, t, PV_QR) + i, qr);
    __stcs(pvec(a, t, PV_QI) + i, qi);
    v[0] = pr[i] * qr - pi[i] * qi;
    v[1] = pr[i] * qi + pi[i] * qr;
  }
  if (ptask_reduce<2>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.td + t * 8;
    const double den = v[0] * v[0] + v[1] * v[1];
    if (!(den > 0.0)) {
      a.ti[t * 4] = 2;                 // breakdown: keep the current X
      atomicAdd(a.counters + 1, 1);
    } else {
      td[3] = (td[0] * v[0] + td[1] * v[1]) / den;
      td[4] = (td[1] * v[0] - td[0] * v[1]) / den;
    }
  }
}

// x += alpha p; r -= alpha q; z = D^-1 r; rho' = r^T z, |r|^2; last block: beta / stop
__global__ void __launch_bounds__(kThreads) pupdate_kernel(PArgs a) {
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  if (!block_uniform(a.ti[t * 4] == 1)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double* td = a.td + t * 8;
  const double ar = td[3], ai = td[4];
  double v[3] = {0.0, 0.0, 0.0};
  if (i < a.N) {
    // every vector is read / written once per launch: streamed (evict first)
    const double pr = __ldcs(pvec(a, t, PV_PR) + i), pi = __ldcs(pvec(a, t, PV_PI) + i);
    const double qr = __ldcs(pvec(a, t, PV_QR) + i), qi = __ldcs(pvec(a, t, PV_QI) + i);
    __stcs(pvec(a, t, PV_XR) + i, __ldcs(pvec(a, t, PV_XR) + i) + (ar * pr - ai * pi));
    __stcs(pvec(a, t, PV_XI) + i, __ldcs(pvec(a, t, PV_XI) + i) + (ar * pi + ai * pr));
    const double rr = __ldcs(pvec(a, t, PV_RR) + i) - (ar * qr - ai * qi);
    const double ri = __ldcs(pvec(a, t, PV_RI) + i) - (ar * qi + ai * qr);
    __stcs(pvec(a, t, PV_RR) + i, rr);
    __stcs(pvec(a, t, PV_RI) + i, ri);
    const double dr = __ldcs(pvec(a, t, PV_DR) + i), di = __ldcs(pvec(a, t, PV_DI) + i);
    const double zr = dr * rr - di * ri, zi = dr * ri + di * rr;
    __stcs(pvec(a, t, PV_ZR) + i, zr);
    __stcs(pvec(a, t, PV_ZI) + i, zi);
    v[0] = rr * zr - ri * zi;
    v[1] = rr * zi + ri * zr;
    v[2] = rr * rr + ri * ri;
  }
  if (ptask_reduce<3>(v, a, t, red) && threadIdx.x == 0) {
    double* tdw = a.td + t * 8;
    int32_t* ti = a.ti + t * 4;
    ti[1] += 1;
    const double rden = tdw[0] * tdw[0] + tdw[1] * tdw[1];
    if (v[2] <= a.rtol2 * tdw[2] || !isfinite(v[2]) || ti[1] >= a.max_it || !(rden > 0.0)) {
      ti[0] = 2;
      atomicAdd(a.counters + 1, 1);
    } else {
      tdw[5] = (v[0] * tdw[0] + v[1] * tdw[1]) / rden;
      tdw[6] = (v[1] * tdw[0] - v[0] * tdw[1]) / rden;
      tdw[0] = v[0];
      tdw[1] = v[1];
    }
  }
}

__global__ void __launch_bounds__(kThreads) ppupd_kernel(PArgs a) {
  const int t = blockIdx.y;
  if (a.ti[t * 4] != 1) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double br = a.td[t * 8 + 5], bi = a.td[t * 8 + 6];
  const double pr = __ldcs(pvec(a, t, PV_PR) + i), pi = __ldcs(pvec(a, t, PV_PI) + i);
  __stcs(pvec(a, t, PV_PR) + i, __ldcs(pvec(a, t, PV_ZR) + i) + (br * pr - bi * pi));
  __stcs(pvec(a, t, PV_PI) + i, __ldcs(pvec(a, t, PV_ZI) + i) + (br * pi + bi * pr));
}

// ---- region-linear variant (config 2: 256^2 blocks8 grids) -----------------
// The same COCG iteration with Z applied from the task's class table: a PCG-
// style launch triple moves read p, write q | read p q x r, write x r | read
// r p, write p = 176 B per point and iteration instead of 336 (no streamed
// M / K values, no stored D^-1 and z).  These launches run next to another
// call's band kernel on the SMs its clusters leave idle (mlmc.run_level_calls),
// so their HBM / L2 traffic is what they cost the estimate.
constexpr int kPTW = 16;   // doubles per class in PArgs::ctab

__global__ void ptab_kernel(PArgs a) {
  __shared__ double2 sp[16];
  const int t = blockIdx.x;
  const int s = a.sample[t];
  if (threadIdx.x < a.R)
    sp[threadIdx.x] = reinterpret_cast<const double2*>(a.rpar)[(int64_t)s * a.R + threadIdx.x];
  __syncthreads();
  double c1, sn, dt;
  item_cs(a, t, c1, sn, dt);
  for (int c = threadIdx.x; c < a.rC; c += blockDim.x) {
    const uint32_t key = __ldg(a.rckey + c);
    const uint32_t code = key & 0x00ffffffu, mask = key >> 24;
    double2 p[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) p[e] = sp[(code >> (4 * e)) & 15u];
    double M7[7], K7[7];
    double m = 0.0, k = 0.0;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      m = __dadd_rn(m, __dmul_rn(p[e].x, a.rmw[e]));
      k = __dadd_rn(k, __dmul_rn(p[e].y, a.rkw[e]));
    }
    M7[3] = m;
    K7[3] = k;
    const int slot[6] = {0, 1, 2, 4, 5, 6};
    const int e0[6] = {0, 0, 1, 2, 3, 4}, e1[6] = {1, 2, 3, 4, 5, 5};
    const int cw[6] = {10, 8, 6, 6, 8, 10};
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const bool ok = (mask >> j) & 1u;
      M7[slot[j]] = ok ? __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[j]].x, a.rmw[cw[j]])),
                                   __dmul_rn(p[e1[j]].x, a.rmw[cw[j] + 1]))
                       : 0.0;
      K7[slot[j]] = ok ? __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[j]].y, a.rkw[cw[j]])),
                                   __dmul_rn(p[e1[j]].y, a.rkw[cw[j] + 1]))
                       : 0.0;
    }
    double* T = a.ctab + ((int64_t)t * a.rC + c) * kPTW;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      T[d] = fma(c1, M7[d], dt * K7[d]);
      T[8 + d] = sn * M7[d];
    }
    const double dr = T[3], di = T[11], den = dr * dr + di * di;
    T[7] = den > 0.0 ? dr / den : 0.0;
    T[15] = den > 0.0 ? -di / den : 0.0;
  }
}

__device__ __forceinline__ void ptab_load(const PArgs& a, int t, double* tab) {
  const double* g = a.ctab + (int64_t)t * a.rC * kPTW;
  for (int i = threadIdx.x; i < a.rC * kPTW; i += blockDim.x) tab[i] = __ldg(g + i);
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) pinit_rg_kernel(PArgs a) {
  extern __shared__ __align__(16) double ptab[];
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  ptab_load(a, t, ptab);
  const double dt = a.dt[t];
  double v[3] = {0.0, 0.0, 0.0};
  if (i < a.N) {
    const double* T = ptab + (int)__ldg(a.rcls + i) * kPTW;
    const double ir = T[7], ii = T[15];
    const double b = dt * a.profile[i];
    pvec(a, t, PV_XR)[i] = 0.0;
    pvec(a, t, PV_XI)[i] = 0.0;
    pvec(a, t, PV_RR)[i] = b;
    pvec(a, t, PV_RI)[i] = 0.0;
    pvec(a, t, PV_PR)[i] = ir * b;
    pvec(a, t, PV_PI)[i] = ii * b;
    v[0] = b * ir * b;
    v[1] = b * ii * b;
    v[2] = b * b;
  }
  if (ptask_reduce<3>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.td + t * 8;
    td[0] = v[0];
    td[1] = v[1];
    td[2] = v[2];
    a.ti[t * 4 + 0] = v[2] > 0.0 ? 1 : 0;
    a.ti[t * 4 + 1] = 0;
    atomicAdd(a.counters + 0, 1);
    if (!(v[2] > 0.0)) atomicAdd(a.counters + 1, 1);
  }
}

__global__ void __launch_bounds__(kThreads) pspmv_rg_kernel(PArgs a) {
  extern __shared__ __align__(16) double ptab[];
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  if (!block_uniform(a.ti[t * 4] == 1)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  ptab_load(a, t, ptab);
  double v[2] = {0.0, 0.0};
  if (i < a.N) {
    const double* T = ptab + (int)__ldg(a.rcls + i) * kPTW;
    const double* pr = pvec(a, t, PV_PR);
    const double* pi = pvec(a, t, PV_PI);
    const int off[7] = {-a.wd - 1, -a.wd, -1, 0, 1, a.wd, a.wd + 1};
    double qr = 0.0, qi = 0.0, pcr = 0.0, pci = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      const double zr = T[d], zi = T[8 + d];
      if (zr != 0.0 || zi != 0.0) {      // a zero coefficient: no such neighbour
        const double xr = pr[i + off[d]], xi = pi[i + off[d]];
        qr = fma(zr, xr, fma(-zi, xi, qr));
        qi = fma(zr, xi, fma(zi, xr, qi));
        if (d == 3) {
          pcr = xr;
          pci = xi;
        }
      }
    }
    __stcs(pvec(a, t, PV_QR) + i, qr);
    __stcs(pvec(a, t, PV_QI) + i, qi);
    v[0] = pcr * qr - pci * qi;
    v[1] = pcr * qi + pci * qr;
  }
  if (ptask_reduce<2>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.td + t * 8;
    const double den = v[0] * v[0] + v[1] * v[1];
    if (!(den > 0.0)) {
      a.ti[t * 4] = 2;
      atomicAdd(a.counters + 1, 1);
    } else {
      td[3] = (td[0] * v[0] + td[1] * v[1]) / den;
      td[4] = (td[1] * v[0] - td[0] * v[1]) / den;
    }
  }
}

__global__ void __launch_bounds__(kThreads) pupdate_rg_kernel(PArgs a) {
  extern __shared__ __align__(16) double ptab[];
  __shared__ double red[2 * 4 * 32];
  const int t = blockIdx.y;
  if (!block_uniform(a.ti[t * 4] == 1)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  ptab_load(a, t, ptab);
  const double* td = a.td + t * 8;
  const double ar = td[3], ai = td[4];
  double v[3] = {0.0, 0.0, 0.0};
  if (i < a.N) {
    const double* T = ptab + (int)__ldg(a.rcls + i) * kPTW;
    const double pr = pvec(a, t, PV_PR)[i], pi = pvec(a, t, PV_PI)[i];
    const double qr = __ldcs(pvec(a, t, PV_QR) + i), qi = __ldcs(pvec(a, t, PV_QI) + i);
    __stcs(pvec(a, t, PV_XR) + i, __ldcs(pvec(a, t, PV_XR) + i) + (ar * pr - ai * pi));
    __stcs(pvec(a, t, PV_XI) + i, __ldcs(pvec(a, t, PV_XI) + i) + (ar * pi + ai * pr));
    const double rr = __ldcs(pvec(a, t, PV_RR) + i) - (ar * qr - ai * qi);
    const double ri = __ldcs(pvec(a, t, PV_RI) + i) - (ar * qi + ai * qr);
    pvec(a, t, PV_RR)[i] = rr;
    pvec(a, t, PV_RI)[i] = ri;
    const double dr = T[7], di = T[15];
    const double zr = dr * rr - di * ri, zi = dr * ri + di * rr;
    v[0] = rr * zr - ri * zi;
    v[1] = rr * zi + ri * zr;
    v[2] = rr * rr + ri * ri;
  }
  if (ptask_reduce<3>(v, a, t, red) && threadIdx.x == 0) {
    double* tdw = a.td + t * 8;
    int32_t* ti = a.ti + t * 4;
    ti[1] += 1;
    const double rden = tdw[0] * tdw[0] + tdw[1] * tdw[1];
    if (v[2] <= a.rtol2 * tdw[2] || !isfinite(v[2]) || ti[1] >= a.max_it || !(rden > 0.0)) {
      ti[0] = 2;
      atomicAdd(a.counters + 1, 1);
    } else {
      tdw[5] = (v[0] * tdw[0] + v[1] * tdw[1]) / rden;
      tdw[6] = (v[1] * tdw[0] - v[0] * tdw[1]) / rden;
      tdw[0] = v[0];
      tdw[1] = v[1];
    }
  }
}

// p = D^-1 r + beta p (z recomputed from r, not stored)
__global__ void __launch_bounds__(kThreads) ppupd_rg_kernel(PArgs a) {
  extern __shared__ __align__(16) double ptab[];
  const int t = blockIdx.y;
  if (!block_uniform(a.ti[t * 4] == 1)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  ptab_load(a, t, ptab);
  if (i >= a.N) return;
  const double* T = ptab + (int)__ldg(a.rcls + i) * kPTW;
  const double br = a.td[t * 8 + 5], bi = a.td[t * 8 + 6];
  const double rr = pvec(a, t, PV_RR)[i], ri = pvec(a, t, PV_RI)[i];
  const double dr = T[7], di = T[15];
  const double zr = dr * rr - di * ri, zi = dr * ri + di * rr;
  const double pr = pvec(a, t, PV_PR)[i], pi = pvec(a, t, PV_PI)[i];
  pvec(a, t, PV_PR)[i] = zr + (br * pr - bi * pi);
  pvec(a, t, PV_PI)[i] = zi + (br * pi + bi * pr);
}

__global__ void pfinal_kernel(PArgs a) {
  const int t = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double xr = pvec(a, t, PV_XR)[i], xi = pvec(a, t, PV_XI)[i];
  const bool fin = isfinite(xr) && isfinite(xi);
  a.X[((int64_t)t * 2) * a.N + i] = fin ? xr : 0.0;
  a.X[((int64_t)t * 2 + 1) * a.N + i] = fin ? xi : 0.0;
}

}  // namespace

size_t stream_workspace_bytes(const Ctx* ctx, int n_tasks, int S) {
  const Layout L = make_layout(ctx, n_tasks, S);
  // the cooperative path reuses the region after A / dinv
  return std::max(L.total, L.off[2] + coop_workspace_bytes(ctx, n_tasks));
}

int stream_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, int S, const double* M,
                     const double* K, const double* rpar, const double* profile, double omega,
                     double rtol,
                     int max_it, const double* xss, double* xbuf, double* qoi, int32_t* iters,
                     int32_t* status, const int32_t* active, int64_t* elapsed, void* ws,
                     size_t ws_bytes, cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  const Layout L = make_layout(ctx, n_tasks, S);
  // the streaming kernels need one dt per call (one operator per sample); the
  // band path forms each task's class table from its own dt and takes any mix
  std::vector<mlmcp_task> h(n_tasks);
  MLMCP_CUDA_CHECK(cudaMemcpyAsync(h.data(), tasks, sizeof(mlmcp_task) * n_tasks,
                                   cudaMemcpyDeviceToHost, stream));
  MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
  int steps_max = 0;
  bool mixed_dt = false;
  for (const auto& t : h) {
    mixed_dt |= t.dt != h[0].dt;
    if (t.sample < 0 || t.sample >= S) {
      set_error("task sample index out of range");
      return MLMCP_EINVAL;
    }
    if (t.qoi_mode == MLMCP_QOI_ELECTRICAL || t.qoi_mode == MLMCP_QOI_JOULE) {
      set_error("streaming path: QoI modes ELECTRICAL / JOULE need the SM-resident or direct path");
      return MLMCP_EINVAL;
    }
    steps_max = std::max(steps_max, t.n_steps);
  }
  bool any_ss = false, any_corr = false;
  for (const auto& t : h) {
    any_ss |= (t.ss_slot >= 0 && !(t.flags & MLMCP_TASK_NO_EXTRAPOLATION));
    any_corr |= (t.flags & MLMCP_TASK_CORRECTION) != 0;
    if ((t.flags & MLMCP_TASK_CORRECTION) && t.qoi_mode != MLMCP_QOI_NONE) {
      set_error("correction tasks (MLMCP_TASK_CORRECTION) carry no QoI");
      return MLMCP_EINVAL;
    }
  }
  const bool band_call = !any_corr && !(cluster_usable(ctx) && !(any_ss && xss != nullptr)) &&
                         band_usable(ctx) && rpar != nullptr && region_on() && ws != nullptr &&
                         ws_bytes >= L.total && band_ring_bytes(n_tasks) <= ws_bytes;
  if (mixed_dt && !band_call) {
    set_error("streaming path: all tasks of one call must share dt");
    return MLMCP_EINVAL;
  }
  if (any_corr) {   // correction solves run on the tile kernels only
    if (!tile_usable(ctx)) {
      set_error("MLMCP_TASK_CORRECTION needs the streaming tile path (structured grid)");
      return MLMCP_EINVAL;
    }
    if (ws == nullptr || ws_bytes < L.total) {
      set_error("streaming workspace too small: need " + std::to_string(L.total) + " bytes");
      return MLMCP_ENOMEM;
    }
    Work w = carve(ws, L);
    SArgs a = make_args(ctx, n_tasks, S, tasks, M, K, profile, omega, rtol, max_it, xbuf, qoi,
                        iters, status, active, w);
    set_region(ctx, a, rpar);
    a.xss = xss;
    return run_steps(ctx, a, steps_max, h[0].dt, stream);
  }
  // one thread-block cluster per task when a sample's grid fits a cluster
  // (cluster_path.cu); it predicts by extrapolation only, so batches that
  // carry periodic steady states stay on the kernels below
  if (cluster_usable(ctx) && !(any_ss && xss != nullptr))
    return cluster_propagate(ctx, n_tasks, tasks, S, M, K, profile, omega, rtol, max_it, xbuf,
                             qoi, iters, status, active, elapsed, ws, ws_bytes, stream);
  if (ws == nullptr || ws_bytes < L.total) {
    set_error("streaming workspace too small: need " + std::to_string(L.total) + " bytes");
    return MLMCP_ENOMEM;
  }
  Work w = carve(ws, L);
  // region-linear grids up to 256 x 256: one 16-CTA cluster per task keeps the
  // PCG vectors on chip (band_path.cu)
  if (band_usable(ctx) && rpar != nullptr && region_on() &&
      band_ring_bytes(n_tasks) <= ws_bytes)   // the band path uses the workspace as its ring
    return band_propagate(ctx, n_tasks, tasks, rpar, profile, omega, rtol, max_it,
                          stream_order(), ls_on(), xss, static_cast<double*>(ws), xbuf, qoi,
                          iters, status, active, elapsed, stream);
  SArgs a = make_args(ctx, n_tasks, S, tasks, M, K, profile, omega, rtol, max_it, xbuf, qoi,
                      iters, status, active, w);
  set_region(ctx, a, rpar);
  a.xss = xss;
  if (coop_usable(ctx, n_tasks) && !(any_ss && xss != nullptr)) {
    // grid-resident path: form the ELL operator once, then one cooperative launch
    // per chunk of tasks runs every step (coop_path.cu)
    const dim3 grid_form((a.N + kThreads - 1) / kThreads, a.S);
    SArgs as = a;                       // stencil-slot layout: slot j <-> offset j
    as.ell_pos = ctx->stencil_pos;
    as.W = ctx->stencil_w;
    as.ell_col = nullptr;
    form_ell_kernel<<<grid_form, kThreads, 0, stream>>>(as, h[0].dt);
    MLMCP_LAUNCH_CHECK("form_ell_kernel(stencil)");
    char* cws = static_cast<char*>(ws) + L.off[2];   // reuse the per-task vector region
    return coop_propagate(ctx, n_tasks, tasks, h, S, w.A, w.dinv, M, K, profile, omega, rtol,
                          max_it, xbuf, qoi, iters, status, active, cws, ws_bytes - L.off[2],
                          stream);
  }
  return run_steps(ctx, a, steps_max, h[0].dt, stream);
}

int stream_path_of(const Ctx* ctx, int n_tasks, int S, bool with_ss, bool with_rp,
                   bool correction) {
  (void)S;
  if (correction) return tile_usable(ctx) ? MLMCP_PATH_TILE : MLMCP_PATH_ELL;
  if (cluster_usable(ctx) && !with_ss) return MLMCP_PATH_CLUSTER;
  if (band_usable(ctx) && with_rp && region_on()) return MLMCP_PATH_BAND;
  if (coop_usable(ctx, n_tasks) && !with_ss) return MLMCP_PATH_COOP;
  return tile_usable(ctx) ? MLMCP_PATH_TILE : MLMCP_PATH_ELL;
}

int stream_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                           const double* rpar, const double* profile, double omega, double dt_c,
                           double t0,
                           const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                           int max_it, double* U, const double* F, double* C, int32_t* iters,
                           int32_t* status, const int32_t* active, void* ws, size_t ws_bytes,
                           cudaStream_t stream) {
  if (S == 0) return MLMCP_OK;
  const int64_t N = ctx->n;
  // workspace: streaming layout for S tasks + tasks[S] + cval[S][N] + tstatus[S][4]
  const Layout L = make_layout(ctx, S, S);
  const size_t tasks_off = L.total;
  const size_t cval_off = tasks_off + align_up(sizeof(mlmcp_task) * S);
  const size_t tst_off = cval_off + align_up(sizeof(double) * S * N);
  const size_t need = tst_off + align_up(sizeof(int32_t) * kStatusInts * S);
  if (ws == nullptr || ws_bytes < need) {
    set_error("streaming workspace too small for the coarse sweep: need " +
              std::to_string(need) + " bytes");
    return MLMCP_ENOMEM;
  }
  char* base = static_cast<char*>(ws);
  mlmcp_task* dtasks = reinterpret_cast<mlmcp_task*>(base + tasks_off);
  double* cval = reinterpret_cast<double*>(base + cval_off);
  int32_t* tstatus = reinterpret_cast<int32_t*>(base + tst_off);
  if (cluster_usable(ctx)) {   // one launch for the whole sweep (cluster_path.cu)
    int32_t* act = const_cast<int32_t*>(active);
    const dim3 grid((unsigned)((N + 255) / 256), S);
    if (k > 1) {
      freeze_kernel<<<grid, 256, 0, stream>>>(S, m, (int)N, k - 1, k - 1, U, F, act);
      MLMCP_LAUNCH_CHECK("freeze_kernel");
    }
    const int rc = cluster_parareal_coarse(ctx, S, k, m, M, K, profile, omega, dt_c, t0,
                                           slice_k0, slice_steps, rtol, max_it, U, F, C, status,
                                           active, stream);
    if (rc != MLMCP_OK) return rc;
    if (k > 1) {
      freeze_kernel<<<grid, 256, 0, stream>>>(S, m, (int)N, m, m, U, F, act);
      MLMCP_LAUNCH_CHECK("freeze_kernel");
    }
    (void)iters;
    return MLMCP_OK;
  }
  std::vector<int64_t> hk0(m);
  std::vector<int32_t> hsteps(m);
  MLMCP_CUDA_CHECK(cudaMemcpyAsync(hk0.data(), slice_k0, sizeof(int64_t) * m,
                                   cudaMemcpyDeviceToHost, stream));
  MLMCP_CUDA_CHECK(cudaMemcpyAsync(hsteps.data(), slice_steps, sizeof(int32_t) * m,
                                   cudaMemcpyDeviceToHost, stream));
  MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
  int32_t* act = const_cast<int32_t*>(active);
  const dim3 grid((unsigned)((N + 255) / 256), S);
  if (k > 1) {
    freeze_kernel<<<grid, 256, 0, stream>>>(S, m, (int)N, k - 1, k - 1, U, F, act);
    MLMCP_LAUNCH_CHECK("freeze_kernel");
  }

  std::vector<mlmcp_task> h(S);
  Work w = carve(ws, L);
  for (int n = k; n < m; ++n) {
    for (int s = 0; s < S; ++s) {
      mlmcp_task& t = h[s];
      t.sample = s;
      t.n_steps = hsteps[n - 1];
      t.k0 = hk0[n - 1];
      t.dt = dt_c;
      t.t_base = t0;
      t.x_in = ((int64_t)s * (m + 1) + (n - 1)) * N;
      t.x_out = -1;
      t.traj = -1;
      t.qoi_slot = -1;
      t.qoi_mode = MLMCP_QOI_NONE;
      t.qoi_from = 0;
      t.group = s;
      t.slot = s;
      t.tag = n;
      t.flags = 0;
      t.qoi_index = 0;
      t.ss_slot = -1;
    }
    MLMCP_CUDA_CHECK(cudaMemcpyAsync(dtasks, h.data(), sizeof(mlmcp_task) * S,
                                     cudaMemcpyHostToDevice, stream));
    MLMCP_CUDA_CHECK(cudaMemsetAsync(tstatus, 0, sizeof(int32_t) * kStatusInts * S, stream));
    // inputs are read from U (x_in); x_out = -1 leaves the terminal states in
    // the work buffer X (task t == sample s), from which cval is taken.
    SArgs a = make_args(ctx, S, S, dtasks, M, K, profile, omega, rtol, max_it, U, nullptr,
                        nullptr, tstatus, act, w);
    set_region(ctx, a, rpar);
    int rc = run_steps(ctx, a, hsteps[n - 1], dt_c, stream);
    if (rc != MLMCP_OK) return rc;
    MLMCP_CUDA_CHECK(cudaMemcpyAsync(cval, w.X, sizeof(double) * S * N,
                                     cudaMemcpyDeviceToDevice, stream));
    coarse_status_kernel<<<(S + 255) / 256, 256, 0, stream>>>(S, k, n, tstatus, status, act);
    MLMCP_LAUNCH_CHECK("coarse_status_kernel");
    correct_kernel<<<grid, 256, 0, stream>>>(S, m, (int)N, n, k, cval, U, F, C, act, status);
    MLMCP_LAUNCH_CHECK("correct_kernel");
  }
  if (k > 1) {
    freeze_kernel<<<grid, 256, 0, stream>>>(S, m, (int)N, m, m, U, F, act);
    MLMCP_LAUNCH_CHECK("freeze_kernel");
  }
  (void)iters;
  return MLMCP_OK;
}

size_t stream_periodic_workspace_bytes(const Ctx* ctx, int n) {
  const size_t N = ctx->n, T = n, nblk = (N + kThreads - 1) / kThreads;
  return align_up(T * kPV * N * 8) + align_up(T * nblk * 4 * 8) + align_up(T * 8 * 8) +
         align_up(T * 4 * 4) + align_up(T * 4) + 64 +
         align_up(T * (size_t)std::max(ctx->rC, 0) * kPTW * 8);
}

int stream_periodic(Ctx* ctx, int n, const int32_t* sample, const double* dt, const double* M,
                    const double* K, const double* rpar, const double* profile, double omega,
                    double rtol, int max_it, double* X, int32_t* iters, void* ws,
                    size_t ws_bytes, cudaStream_t stream) {
  if (n == 0) return MLMCP_OK;
  const size_t need = stream_periodic_workspace_bytes(ctx, n);
  if (ws == nullptr || ws_bytes < need) {
    set_error("steady-state workspace too small: need " + std::to_string(need) + " bytes");
    return MLMCP_ENOMEM;
  }
  PArgs a{};
  a.T = n;
  a.N = ctx->n;
  a.nblk = (ctx->n + kThreads - 1) / kThreads;
  a.nnz = ctx->nnz;
  a.row_ptr = ctx->row_ptr;
  a.col = ctx->col;
  a.sample = sample;
  a.dt = dt;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.X = X;
  char* b = static_cast<char*>(ws);
  const size_t N = ctx->n, T = n, nblk = a.nblk;
  a.vec = reinterpret_cast<double*>(b);
  b += align_up(T * kPV * N * 8);
  a.partial = reinterpret_cast<double*>(b);
  b += align_up(T * nblk * 4 * 8);
  a.td = reinterpret_cast<double*>(b);
  b += align_up(T * 8 * 8);
  a.ti = reinterpret_cast<int32_t*>(b);
  b += align_up(T * 4 * 4);
  a.arrive = reinterpret_cast<int32_t*>(b);
  b += align_up(T * 4);
  a.counters = reinterpret_cast<int32_t*>(b);
  b += 64;
  // region-linear grids: Z from per-class stencil tables (MLMCP_PERIODIC_REGION=0:
  // the streamed CSR values, A/B)
  const char* pe = getenv("MLMCP_PERIODIC_REGION");
  const bool rg = rpar != nullptr && ctx->rcls != nullptr && ctx->rC > 0 && region_on() &&
                  ctx->cl_wd > 0 && !(pe && atoi(pe) == 0);
  size_t tab_smem = 0;
  if (rg) {
    a.rcls = ctx->rcls;
    a.rckey = ctx->rckey;
    a.rC = ctx->rC;
    a.R = ctx->rR;
    a.wd = ctx->cl_wd;
    a.rpar = rpar;
    for (int i = 0; i < 12; ++i) {
      a.rmw[i] = ctx->rmw[i];
      a.rkw[i] = ctx->rkw[i];
    }
    a.ctab = reinterpret_cast<double*>(b);
    tab_smem = sizeof(double) * kPTW * (size_t)a.rC;
  }
  MLMCP_CUDA_CHECK(cudaMemsetAsync(a.arrive, 0, sizeof(int32_t) * T, stream));
  MLMCP_CUDA_CHECK(cudaMemsetAsync(a.counters, 0, 2 * sizeof(int32_t), stream));
  const dim3 grid((a.N + kThreads - 1) / kThreads, n);
  if (rg) {
    ptab_kernel<<<n, 64, 0, stream>>>(a);
    MLMCP_LAUNCH_CHECK("ptab_kernel");
    pinit_rg_kernel<<<grid, kThreads, tab_smem, stream>>>(a);
    MLMCP_LAUNCH_CHECK("pinit_rg_kernel");
  } else {
    pinit_kernel<<<grid, kThreads, 0, stream>>>(a);
    MLMCP_LAUNCH_CHECK("pinit_kernel");
  }
  int32_t* hc = ctx->host_counters;
  int done_iters = 0;
  while (done_iters < max_it) {
    const int chunk = done_iters == 0 ? 16 : 4;
    for (int c = 0; c < chunk; ++c) {
      if (rg) {
        pspmv_rg_kernel<<<grid, kThreads, tab_smem, stream>>>(a);
        MLMCP_LAUNCH_CHECK("pspmv_rg_kernel");
        pupdate_rg_kernel<<<grid, kThreads, tab_smem, stream>>>(a);
        MLMCP_LAUNCH_CHECK("pupdate_rg_kernel");
        ppupd_rg_kernel<<<grid, kThreads, tab_smem, stream>>>(a);
        MLMCP_LAUNCH_CHECK("ppupd_rg_kernel");
        continue;
      }
      pspmv_kernel<<<grid, kThreads, 0, stream>>>(a);
      MLMCP_LAUNCH_CHECK("pspmv_kernel");
      pupdate_kernel<<<grid, kThreads, 0, stream>>>(a);
      MLMCP_LAUNCH_CHECK("pupdate_kernel");
      ppupd_kernel<<<grid, kThreads, 0, stream>>>(a);
      MLMCP_LAUNCH_CHECK("ppupd_kernel");
    }
    done_iters += chunk;
    MLMCP_CUDA_CHECK(cudaMemcpyAsync(hc, a.counters, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                     stream));
    MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (hc[1] >= hc[0]) break;
  }
  pfinal_kernel<<<grid, kThreads, 0, stream>>>(a);
  MLMCP_LAUNCH_CHECK("pfinal_kernel");
  (void)iters;
  return MLMCP_OK;
}

}  // namespace mlmcp
