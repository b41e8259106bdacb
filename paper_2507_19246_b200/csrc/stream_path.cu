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

constexpr int kRingS = 4;   // past states a_{n-1..n-4} (order <= 4 extrapolation)

struct Work {
  double* ring;    // [kRingS][T][N]
  double* A;       // [S][W][N]
  double* dinv;    // [S][N]
  double* X;       // [T][N]
  double* R;
  double* P;
  double* Sv;
  double* Wv;
  double* partial; // [T][nblk][4]
  double* td;      // [T][kTD]
  int32_t* ti;     // [T][kTI]
  int32_t* arrive; // [T]
  int32_t* counters;  // [0] live, [1] done
};

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t off[13];
  size_t total;
};

Layout make_layout(const Ctx* ctx, int T, int S) {
  // operator slots: ELL width, or the stencil width for the cooperative path
  const size_t N = ctx->n, W = std::max(ctx->max_row_nnz, ctx->stencil_w), T_ = T, S_ = S;
  const size_t nblk = (N + kThreads - 1) / kThreads;
  size_t sizes[13] = {S_ * W * N * 8, S_ * N * 8, T_ * N * 8, T_ * N * 8, T_ * N * 8,
                      T_ * N * 8,     T_ * N * 8, T_ * nblk * 4 * 8, T_ * kTD * 8,
                      T_ * kTI * 4,   T_ * 4,     64, kRingS * T_ * N * 8};
  Layout L;
  size_t o = 0;
  for (int i = 0; i < 13; ++i) {
    L.off[i] = o;
    o += align_up(sizes[i]);
  }
  L.total = o;
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
  Work w;
};

// Block reduce of NV values to thread 0, then the last-arriving block of the
// task reduces all partials in fixed order.  Returns true in the last block
// (all threads), with totals in v.
template <int NV>
__device__ __forceinline__ bool task_reduce(double (&v)[NV], const SArgs& a, int t,
                                            double* red) {
  __shared__ bool last;
  int par = 0;
  block_allsum<NV>(v, red, par);
  if (threadIdx.x == 0) {
    double* dst = a.w.partial + ((int64_t)t * a.nblk + blockIdx.x) * 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) dst[k] = v[k];
    __threadfence();
    const int prev = atomicAdd(a.w.arrive + t, 1);
    last = (prev == a.nblk - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < a.nblk; b += blockDim.x) {
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
__global__ void __launch_bounds__(kThreads) guess_kernel(SArgs a, int step) {
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
  const int pmax = pred ? 3 : kRingS;
  const int p = (tk.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : min(step, pmax);
  auto past = [&](int k) { return a.w.ring[(int64_t)((step - k) & (kRingS - 1)) * TN + o]; };
  double g = yn;
  if (p == 1) g = fma(2.0, yn, -past(1));
  else if (p == 2) g = fma(3.0, yn - past(1), past(2));
  else if (p == 3) g = fma(4.0, yn + past(2), fma(-6.0, past(1), -past(3)));
  else if (p >= 4) g = fma(5.0, yn - past(3), fma(10.0, past(2) - past(1), past(4)));
  a.w.ring[(int64_t)(step & (kRingS - 1)) * TN + o] = yn;
  a.w.Wv[o] = an;
  a.w.X[o] = g + sst;
}

// rhs b = M a_n + dt*sf*prof, r = b - A x0, partial b.D^-1.b (Jacobi-weighted
// norm of the stopping rule, as the SM-resident path)
__global__ void __launch_bounds__(kThreads) step_init_kernel(SArgs a, int step) {
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
    for (int j = 0; j < a.W; ++j)
      ax = fma(As[(int64_t)j * a.N + i], X[a.ell_col[j * a.N + i]], ax);
    const double b = __dadd_rn(mx, __dmul_rn(tk.dt, __dmul_rn(sf, a.profile[i])));
    a.w.R[(int64_t)t * a.N + i] = b - ax;
    bb = b * a.w.dinv[(int64_t)s * a.N + i] * b;
  }
  double v[1] = {bb};
  if (task_reduce<1>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.w.td + t * kTD;
    int32_t* ti = a.w.ti + t * kTI;
    td[D_BB] = v[0];
    ti[I_IT_STEP] = 0;
    ti[I_FIRST] = 1;
    atomicAdd(a.w.counters + 0, 1);
    if (v[0] == 0.0) {
      ti[I_STATE] = ST_ZERO;
      atomicAdd(a.w.counters + 1, 1);
    } else {
      ti[I_STATE] = ST_RUN;
    }
  }
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
  if (task_reduce<3>(v, a, t, red) && threadIdx.x == 0) {
    double* td = a.w.td + t * kTD;
    int32_t* ti = a.w.ti + t * kTI;
    const double gamma = v[0], delta = v[1];
    int code = MLMCP_ST_OK;
    bool stop = false;
    if (gamma <= a.rtol2 * td[D_BB]) {   // r.D^-1.r <= rtol^2 b.D^-1.b
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
      atomicAdd(a.w.counters + 1, 1);
    } else {
      ti[I_FIRST] = (ti[I_IT_STEP] == 0);
      ti[I_IT_STEP] += 1;
      ti[I_IT_TOTAL] += 1;
    }
  }
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

// mode 0: per-step (trajectory store + SUM_ENERGY accumulation);
// mode 1: finalize (x_out, FINAL_ENERGY / SUM write-out, iters, status)
__global__ void __launch_bounds__(kThreads) step_end_kernel(SArgs a, int step, int mode) {
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
    const int64_t g = tk.k0 + step + 1;
    energy = tk.qoi_mode == MLMCP_QOI_SUM_ENERGY && g > tk.qoi_from && tk.qoi_slot >= 0;
  } else {
    if (tk.x_out >= 0 && i < a.N) a.xbuf[tk.x_out + i] = X[i];
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
__global__ void mark_fail_kernel(SArgs a, int step) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  int32_t* ti = a.w.ti + t * kTI;
  if (ti[I_CODE] != MLMCP_ST_OK && ti[I_FAILSTEP] < 0) ti[I_FAILSTEP] = step;
  if (ti[I_CODE] == MLMCP_ST_OK) ti[I_FAILSTEP] = -1;
}

int run_steps(Ctx* ctx, SArgs& a, int n_steps_max, double dt, cudaStream_t stream) {
  const dim3 blk(kThreads);
  const dim3 grid_rows((a.N + kThreads - 1) / kThreads, a.T);
  const dim3 grid_form((a.N + kThreads - 1) / kThreads, a.S);
  form_ell_kernel<<<grid_form, blk, 0, stream>>>(a, dt);
  MLMCP_LAUNCH_CHECK("form_ell_kernel");
  copy_in_kernel<<<grid_rows, blk, 0, stream>>>(a);
  MLMCP_LAUNCH_CHECK("copy_in_kernel");
  mark_fail_kernel<<<(a.T + 255) / 256, 256, 0, stream>>>(a, 0);
  MLMCP_LAUNCH_CHECK("mark_fail_kernel");
  int32_t* hc = ctx->host_counters;
  int chunk = 4;
  for (int step = 0; step < n_steps_max; ++step) {
    MLMCP_CUDA_CHECK(cudaMemsetAsync(a.w.counters, 0, 2 * sizeof(int32_t), stream));
    guess_kernel<<<grid_rows, blk, 0, stream>>>(a, step);
    MLMCP_LAUNCH_CHECK("guess_kernel");
    step_init_kernel<<<grid_rows, blk, 0, stream>>>(a, step);
    MLMCP_LAUNCH_CHECK("step_init_kernel");
    int done_iters = 0;
    for (;;) {
      for (int c = 0; c < chunk; ++c) {
        spmv_kernel<<<grid_rows, blk, 0, stream>>>(a);
        MLMCP_LAUNCH_CHECK("spmv_kernel");
        update_kernel<<<grid_rows, blk, 0, stream>>>(a);
        MLMCP_LAUNCH_CHECK("update_kernel");
      }
      done_iters += chunk;
      MLMCP_CUDA_CHECK(cudaMemcpyAsync(hc, a.w.counters, 2 * sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, stream));
      MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
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
  a.w = w;
  return a;
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
      mr = fma(Ms[q], xr, mr);
      mi = fma(Ms[q], xi, mi);
      kr = fma(Ks[q], xr, kr);
      ki = fma(Ks[q], xi, ki);
    }
    // Zr p = c1 M p + dt K p;  Zi p = sn M p;  q = Zr p + i Zi p
    const double zr_r = fma(c1, mr, dt * kr), zr_i = fma(c1, mi, dt * ki);
    const double qr = zr_r - sn * mi, qi = zr_i + sn * mr;
    pvec(a, t, PV_QR)[i] = qr;
    pvec(a, t, PV_QI)[i] = qi;
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
    const double pr = pvec(a, t, PV_PR)[i], pi = pvec(a, t, PV_PI)[i];
    const double qr = pvec(a, t, PV_QR)[i], qi = pvec(a, t, PV_QI)[i];
    pvec(a, t, PV_XR)[i] += ar * pr - ai * pi;
    pvec(a, t, PV_XI)[i] += ar * pi + ai * pr;
    const double rr = pvec(a, t, PV_RR)[i] - (ar * qr - ai * qi);
    const double ri = pvec(a, t, PV_RI)[i] - (ar * qi + ai * qr);
    pvec(a, t, PV_RR)[i] = rr;
    pvec(a, t, PV_RI)[i] = ri;
    const double dr = pvec(a, t, PV_DR)[i], di = pvec(a, t, PV_DI)[i];
    const double zr = dr * rr - di * ri, zi = dr * ri + di * rr;
    pvec(a, t, PV_ZR)[i] = zr;
    pvec(a, t, PV_ZI)[i] = zi;
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
  const double pr = pvec(a, t, PV_PR)[i], pi = pvec(a, t, PV_PI)[i];
  pvec(a, t, PV_PR)[i] = pvec(a, t, PV_ZR)[i] + (br * pr - bi * pi);
  pvec(a, t, PV_PI)[i] = pvec(a, t, PV_ZI)[i] + (br * pi + bi * pr);
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
                     const double* K, const double* profile, double omega, double rtol,
                     int max_it, const double* xss, double* xbuf, double* qoi, int32_t* iters,
                     int32_t* status, const int32_t* active, int64_t* elapsed, void* ws,
                     size_t ws_bytes, cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  const Layout L = make_layout(ctx, n_tasks, S);
  // the streaming path needs one dt per call (one ELL operator per sample)
  std::vector<mlmcp_task> h(n_tasks);
  MLMCP_CUDA_CHECK(cudaMemcpyAsync(h.data(), tasks, sizeof(mlmcp_task) * n_tasks,
                                   cudaMemcpyDeviceToHost, stream));
  MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
  int steps_max = 0;
  for (const auto& t : h) {
    if (t.dt != h[0].dt) {
      set_error("streaming path: all tasks of one call must share dt");
      return MLMCP_EINVAL;
    }
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
  bool any_ss = false;
  for (const auto& t : h) any_ss |= (t.ss_slot >= 0 && !(t.flags & MLMCP_TASK_NO_EXTRAPOLATION));
  // one thread-block cluster per task when a sample's grid fits a cluster
  // (cluster_path.cu); it predicts by extrapolation only, so batches that
  // carry periodic steady states stay on the kernels below
  if (cluster_usable(ctx) && !(any_ss && xss != nullptr))
    return cluster_propagate(ctx, n_tasks, tasks, M, K, profile, omega, rtol, max_it, xbuf, qoi,
                             iters, status, active, elapsed, stream);
  if (ws == nullptr || ws_bytes < L.total) {
    set_error("streaming workspace too small: need " + std::to_string(L.total) + " bytes");
    return MLMCP_ENOMEM;
  }
  Work w = carve(ws, L);
  SArgs a = make_args(ctx, n_tasks, S, tasks, M, K, profile, omega, rtol, max_it, xbuf, qoi,
                      iters, status, active, w);
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

int stream_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                           const double* profile, double omega, double dt_c, double t0,
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
         align_up(T * 4 * 4) + align_up(T * 4) + 64;
}

int stream_periodic(Ctx* ctx, int n, const int32_t* sample, const double* dt, const double* M,
                    const double* K, const double* profile, double omega, double rtol,
                    int max_it, double* X, int32_t* iters, void* ws, size_t ws_bytes,
                    cudaStream_t stream) {
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
  MLMCP_CUDA_CHECK(cudaMemsetAsync(a.arrive, 0, sizeof(int32_t) * T, stream));
  MLMCP_CUDA_CHECK(cudaMemsetAsync(a.counters, 0, 2 * sizeof(int32_t), stream));
  const dim3 grid((a.N + kThreads - 1) / kThreads, n);
  pinit_kernel<<<grid, kThreads, 0, stream>>>(a);
  MLMCP_LAUNCH_CHECK("pinit_kernel");
  int32_t* hc = ctx->host_counters;
  int done_iters = 0;
  while (done_iters < max_it) {
    const int chunk = done_iters == 0 ? 16 : 4;
    for (int c = 0; c < chunk; ++c) {
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
