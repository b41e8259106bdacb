// coop_path.cu — grid-resident batched implicit Euler for meshes that do not fit
// one SM (128^2 .. 512^2: configs 2, 3, 4).
//
// One cooperative launch (grid = #SMs x 1 CTA of 256 threads) runs every step of
// a batch of tasks (reference: timeint.py:88-128).  The (task, row) pairs of the
// batch are spread over all threads: thread j of CTA b owns R slots
// g = (b*R + r)*256 + j, i.e. R rows of (usually) one task, and keeps their x,
// r, p, s and D^-1 in REGISTERS for the whole solve.  Per PCG iteration only
// the per-sample ELL operator streams from HBM (8 W N bytes) and u is exchanged
// through a global buffer that stays in L2 (8 N written, neighbours re-read):
// ~64 N + 8 W N bytes instead of the ~160 N of a two-launch iteration.
// Per iteration: publish u -> grid barrier -> w = A u + partial dots -> grid
// barrier -> every CTA reduces the partials of every task in a fixed order
// (deterministic, identical in all CTAs) -> alpha/beta/convergence -> update.
// PCG is the same Chronopoulos-Gear Jacobi-PCG with the same extrapolated
// initial guesses (state ring in global memory, touched once per step) and the
// same stopping rule as the SM-resident path.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "mlmcp_internal.cuh"

namespace cg = cooperative_groups;

namespace mlmcp {
namespace {

constexpr int kCoopThreads = 256;
constexpr int kCoopOrder = 4;   // extrapolation order (as the SM-resident path)

struct CoopArgs {
  int T;            // tasks in this launch
  int N;            // rows per task
  int W;            // ELL width
  int R;            // slots per thread (runtime copy of the template)
  int S;            // samples in the A/dinv arrays
  int nb_task;      // max CTAs a task spans (partials per task)
  const mlmcp_task* tasks;
  const double* A;        // [S][W][N]
  const double* dinv;     // [S][N]
  const int32_t* ell_col; // [W][N]
  const int32_t* row_ptr;
  const int32_t* col;
  const double* M;
  const double* K;
  int64_t nnz;
  const double* profile;
  double omega, rtol2;
  int max_it;
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  int32_t* active;
  double* Xb;       // [T][N] exchange: a_n (and the energy)
  double* Gb;       // [T][N] exchange: initial guess
  double* Ub;       // [T][N] exchange: u
  double* ring;     // [kCoopOrder][T][N] state history
  double* part;     // [T][nb_task][4] per-CTA partial sums
  int32_t* first_blk;  // [T] first CTA of task t
  int32_t* n_blk;      // [T] CTAs of task t
  unsigned int* bar;   // grid barrier words: [0] release, [1 + b] flag of CTA b
  unsigned int epoch0; // epoch the words hold at launch
  int off[kMaxNz];     // stencil offsets (col - row) of the operator slots
  int pad;             // zero rows before / after each task's exchange vector
  int ld;              // exchange-vector stride per task = N + 2*pad
};

// per-task state kept (identically) by every CTA in shared memory
struct TaskState {
  double tol2, inv_g, c, alpha, beta;
  int it_step, it_total, code, fail_step, order;
  int done;   // converged for this step, or idle
  int live;   // task still running (not failed / inactive)
  int zero;   // b == 0 this step: a_{n+1} = 0
};

// Grid barrier (all CTAs are co-resident: cooperative launch).  CTA b
// publishes the barrier epoch in flag[b]; CTA 0 gathers every flag with all
// its threads and releases the epoch word the other CTAs spin on (1.7 us on
// 148 SMs vs 2.5 us for a single-counter barrier, scripts/barrier_probe.cu).
// Fences order the exchange-buffer writes before / reads after it (readers
// use ld.cg).  `epoch` counts barriers since the launch (uniform in all CTAs);
// the words start at `base` (monotone across launches).
struct GridBar {
  unsigned int* flags;   // [gridDim.x]
  unsigned int* release;
  unsigned int epoch;
};

__device__ __forceinline__ void grid_barrier(GridBar& gb) {
  const unsigned int e = ++gb.epoch;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    reinterpret_cast<volatile unsigned int*>(gb.flags)[blockIdx.x] = e;
  }
  if (blockIdx.x == 0) {
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      while (reinterpret_cast<volatile unsigned int*>(gb.flags)[b] != e) {
      }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      *reinterpret_cast<volatile unsigned int*>(gb.release) = e;
    }
  } else if (threadIdx.x == 0) {
    while (*reinterpret_cast<volatile unsigned int*>(gb.release) != e) {
    }
  }
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
}

template <int R>
struct Slots {
  int task[R];
  int row[R];
  double x[R], r[R], p[R], s[R], dinv[R];
};

__device__ __forceinline__ int slot_g(int r, int R) {
  return (blockIdx.x * R + r) * kCoopThreads + threadIdx.x;
}

// CTA-wide sum of NV values for the (at most two) tasks of this CTA:
// v_lo/v_hi -> thread 0 writes part[task][blk - first]
template <int NV>
__device__ void cta_partials(double (&lo)[NV], double (&hi)[NV], int t_lo, int t_hi,
                             const CoopArgs& a, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      lo[k] += __shfl_xor_sync(0xffffffffu, lo[k], off);
      hi[k] += __shfl_xor_sync(0xffffffffu, hi[k], off);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      red[warp * 8 + k] = lo[k];
      red[warp * 8 + 4 + k] = hi[k];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * NV) {
    const int half = threadIdx.x / NV, k = threadIdx.x % NV;
    double s = 0.0;
    for (int w = 0; w < kCoopThreads / 32; ++w) s += red[w * 8 + half * 4 + k];  // fixed order
    const int t = half ? t_hi : t_lo;
    if (t >= 0 && (half == 0 || t_hi != t_lo)) {
      const int j = blockIdx.x - a.first_blk[t];
      a.part[((int64_t)t * a.nb_task + j) * 4 + k] = s;
    }
  }
  __syncthreads();
}

// totals[t][k] = sum_j part[t][j][k] in a fixed order (every CTA computes the
// same): warp w reduces tasks w, w+8, ...; lane l sums partials l, l+32, ...
// sequentially, then a fixed xor butterfly.
template <int NV>
__device__ void task_totals(const CoopArgs& a, double* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = warp; t < a.T; t += kCoopThreads / 32) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    const int nb = a.n_blk[t];
    for (int j = lane; j < nb; j += 32) {
      const double* p = a.part + ((int64_t)t * a.nb_task + j) * 4;
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += __ldcg(p + k);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) tot[t * 4 + k] = s[k];
    }
  }
  __syncthreads();
}

// y = A v for slot r from the exchange buffer `buf`: operator in stencil-slot
// layout A[s][j][i] (coefficient of offset off[j], 0 if absent), neighbour
// addresses computed (no column loads); padded buffers absorb the boundary.
template <int R, int W>
__device__ __forceinline__ double sten_apply(const CoopArgs& a, const Slots<R>& sl, int r,
                                             const double* buf) {
  const int t = sl.task[r], i = sl.row[r];
  const double* As = a.A + (int64_t)a.tasks[t].sample * W * a.N + i;
  const double* v = buf + (int64_t)t * a.ld + a.pad + i;
  double av[W], vv[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    av[j] = __ldg(As + (int64_t)j * a.N);
    vv[j] = __ldcg(v + a.off[j]);
  }
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) acc = fma(av[j], vv[j], acc);
  return acc;
}

__device__ __forceinline__ double* xrow(const CoopArgs& a, double* buf, int t, int i) {
  return buf + (int64_t)t * a.ld + a.pad + i;
}

// y = B v for slot r with B given by per-sample CSR values (M or K)
template <int R>
__device__ __forceinline__ double csr_apply(const CoopArgs& a, const Slots<R>& sl, int r,
                                            const double* vals, const double* buf) {
  const int t = sl.task[r], i = sl.row[r];
  const double* Bs = vals + (int64_t)a.tasks[t].sample * a.nnz;
  const double* v = buf + (int64_t)t * a.ld + a.pad;
  double acc = 0.0;
  for (int q = __ldg(a.row_ptr + i); q < __ldg(a.row_ptr + i + 1); ++q)
    acc = fma(__ldg(Bs + q), __ldcg(v + __ldg(a.col + q)), acc);
  return acc;
}

template <int R, int W>
__global__ void __launch_bounds__(kCoopThreads, 1) coop_kernel(CoopArgs a) {
  extern __shared__ __align__(16) double csm[];
  double* red = csm;                         // [8 warps][8]
  double* tot = csm + 64;                    // [T][4]
  TaskState* ts = reinterpret_cast<TaskState*>(csm + 64 + 4 * a.T);
  const int TN = a.T * a.N;
  GridBar gb{a.bar + 1, a.bar, a.epoch0};
  Slots<R> sl;
  int t_lo = -1, t_hi = -1;
  {
    const int g0 = slot_g(0, R) - threadIdx.x;                    // CTA's first slot
    const int g1 = g0 + R * kCoopThreads - 1;
    t_lo = g0 < TN ? g0 / a.N : -1;
    t_hi = g1 < TN ? g1 / a.N : (TN > g0 ? (TN - 1) / a.N : -1);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int g = slot_g(r, R);
    const bool ok = g < TN;
    sl.task[r] = ok ? g / a.N : -1;
    sl.row[r] = ok ? g % a.N : 0;
    sl.x[r] = sl.r[r] = sl.p[r] = sl.s[r] = 0.0;
    sl.dinv[r] = 0.0;
    if (ok) {
      const mlmcp_task& tk = a.tasks[sl.task[r]];
      sl.dinv[r] = a.dinv[(int64_t)tk.sample * a.N + sl.row[r]];
      sl.x[r] = a.xbuf[tk.x_in + sl.row[r]];
      if (tk.traj >= 0) a.xbuf[tk.traj + sl.row[r]] = sl.x[r];
    }
  }
  for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
    const mlmcp_task& tk = a.tasks[t];
    TaskState z{};
    z.live = (a.active == nullptr || tk.group < 0 || a.active[tk.group] != 0) ? 1 : 0;
    z.code = MLMCP_ST_OK;
    ts[t] = z;
  }
  __syncthreads();
  int max_steps = 0;
  for (int t = 0; t < a.T; ++t) max_steps = max(max_steps, a.tasks[t].n_steps);

  for (int step = 0; step < max_steps; ++step) {
    // ---- step start: a_n -> Xb, extrapolated guess -> Gb (ring: a_{n-1..n-4})
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      if (t < 0) continue;
      const int i = sl.row[r];
      const TaskState& st = ts[t];
      const int64_t o = (int64_t)t * a.N + i;
      const double an = sl.x[r];
      *xrow(a, a.Xb, t, i) = an;
      const bool run = st.live && step < a.tasks[t].n_steps;
      const int p = (!run || (a.tasks[t].flags & MLMCP_TASK_NO_EXTRAPOLATION)) ? 0
                                                                             : min(st.order, kCoopOrder);
      auto past = [&](int k) { return a.ring[(int64_t)((step - k) & (kCoopOrder - 1)) * TN + o]; };
      double gss = an;
      if (p == 1) gss = fma(2.0, an, -past(1));
      else if (p == 2) gss = fma(3.0, an - past(1), past(2));
      else if (p == 3) gss = fma(4.0, an + past(2), fma(-6.0, past(1), -past(3)));
      else if (p >= 4) gss = fma(5.0, an - past(3), fma(10.0, past(2) - past(1), past(4)));
      *xrow(a, a.Gb, t, i) = gss;
      sl.x[r] = gss;
    }
    grid_barrier(gb);
    // ---- b = M a_n + dt sf prof, r = b - A x0, u = D r
    double lo4[4] = {0, 0, 0, 0}, hi4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      double res = 0.0, u = 0.0;
      if (t >= 0 && ts[t].live && step < a.tasks[t].n_steps) {
        const mlmcp_task& tk = a.tasks[t];
        const int i = sl.row[r];
        const double sf = sin(__dmul_rn(a.omega, grid_time(tk.t_base, tk.k0 + step + 1, tk.dt)));
        const double mx = csr_apply(a, sl, r, a.M, a.Xb);
        const double ax = sten_apply<R, W>(a, sl, r, a.Gb);
        const double b = __dadd_rn(mx, __dmul_rn(tk.dt, __dmul_rn(sf, __ldg(a.profile + i))));
        res = b - ax;
        u = sl.dinv[r] * res;
        double* acc = (t == t_lo) ? lo4 : hi4;
        acc[3] += b * sl.dinv[r] * b;          // Jacobi-weighted norm of b
      }
      sl.r[r] = res;
      if (t >= 0) *xrow(a, a.Ub, t, sl.row[r]) = u;
    }
    grid_barrier(gb);
    // first SpMV: w = A u; gamma, delta, rho, bb
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      if (t < 0 || !ts[t].live || step >= a.tasks[t].n_steps) continue;
      const double u = sl.dinv[r] * sl.r[r];
      const double w = sten_apply<R, W>(a, sl, r, a.Ub);
      double* acc = (t == t_lo) ? lo4 : hi4;
      acc[0] += sl.r[r] * u;
      acc[1] += w * u;
      acc[2] += sl.r[r] * sl.r[r];
      sl.p[r] = u;
      sl.s[r] = w;
    }
    cta_partials<4>(lo4, hi4, t_lo, t_hi, a, red);
    grid_barrier(gb);
    task_totals<4>(a, tot);
    // decide per task (identical in every CTA); a block-local copy of the state
    for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
      TaskState& st = ts[t];
      st.done = 1;
      st.zero = 0;
      st.it_step = 0;
      if (!st.live || step >= a.tasks[t].n_steps) continue;
      const double gamma = tot[t * 4 + 0], delta = tot[t * 4 + 1], rho = tot[t * 4 + 2];
      const double bb = tot[t * 4 + 3];
      st.tol2 = a.rtol2 * bb;
      if (bb == 0.0) { st.zero = 1; continue; }          // b == 0 exactly: a = 0
      if (gamma <= st.tol2) continue;                     // r.D^-1.r <= rtol^2 b.D^-1.b
      if (!isfinite(gamma) || !isfinite(rho)) { st.code = MLMCP_ST_NONFINITE; st.fail_step = step; st.live = 0; continue; }
      if (!(delta > 0.0)) { st.code = MLMCP_ST_BREAKDOWN; st.fail_step = step; st.live = 0; continue; }
      st.done = 0;
      st.inv_g = fast_rcp(gamma);
      st.c = st.inv_g * (delta * st.inv_g);
      st.alpha = gamma * fast_rcp(delta);                  // first update: p = u, s = w
      st.it_step = 1;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      if (t < 0) continue;
      const TaskState& st = ts[t];
      if (st.zero) { sl.x[r] = 0.0; continue; }
      if (st.done) continue;
      sl.x[r] = fma(st.alpha, sl.p[r], sl.x[r]);
      sl.r[r] = fma(-st.alpha, sl.s[r], sl.r[r]);
    }
    // ---- PCG iterations until every task of the batch converged
    for (;;) {
      bool any = false;
      for (int t = 0; t < a.T; ++t) any |= (ts[t].done == 0);
      if (!any) break;
      double lo3[3] = {0, 0, 0}, hi3[3] = {0, 0, 0};
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = sl.task[r];
        if (t < 0) continue;
        *xrow(a, a.Ub, t, sl.row[r]) = ts[t].done ? 0.0 : sl.dinv[r] * sl.r[r];
      }
      grid_barrier(gb);
      double wv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = sl.task[r];
        wv[r] = 0.0;
        if (t < 0 || ts[t].done) continue;
        const double u = sl.dinv[r] * sl.r[r];
        wv[r] = sten_apply<R, W>(a, sl, r, a.Ub);
        double* acc = (t == t_lo) ? lo3 : hi3;
        acc[0] += sl.r[r] * u;
        acc[1] += wv[r] * u;
        acc[2] += sl.r[r] * sl.r[r];
      }
      double lo4b[4] = {lo3[0], lo3[1], lo3[2], 0.0}, hi4b[4] = {hi3[0], hi3[1], hi3[2], 0.0};
      cta_partials<4>(lo4b, hi4b, t_lo, t_hi, a, red);
      grid_barrier(gb);
      task_totals<3>(a, tot);
      for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
        TaskState& st = ts[t];
        if (st.done) continue;
        const double gnew = tot[t * 4 + 0], delta = tot[t * 4 + 1], rho = tot[t * 4 + 2];
        if (gnew <= st.tol2) { st.done = 1; continue; }
        if (!isfinite(gnew) || !isfinite(rho)) { st.code = MLMCP_ST_NONFINITE; st.fail_step = step; st.live = 0; st.done = 1; continue; }
        if (st.it_step >= a.max_it) { st.code = MLMCP_ST_NOCONV; st.fail_step = step; st.live = 0; st.done = 1; continue; }
        const double beta = gnew * st.inv_g;
        const double den = fma(-(gnew * gnew), st.c, delta);
        if (!(den > 0.0)) { st.code = MLMCP_ST_BREAKDOWN; st.fail_step = step; st.live = 0; st.done = 1; continue; }
        st.alpha = gnew * fast_rcp(den);
        st.beta = beta;
        st.inv_g = fast_rcp(gnew);
        st.c = st.inv_g * (den * st.inv_g);
        st.it_step += 1;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = sl.task[r];
        if (t < 0 || ts[t].done) continue;
        const double alpha = ts[t].alpha, beta = ts[t].beta;
        sl.p[r] = fma(beta, sl.p[r], sl.dinv[r] * sl.r[r]);
        sl.s[r] = fma(beta, sl.s[r], wv[r]);
        sl.x[r] = fma(alpha, sl.p[r], sl.x[r]);
        sl.r[r] = fma(-alpha, sl.s[r], sl.r[r]);
      }
    }
    // ---- end of step: iteration counts, history ring, trajectory, energy
    for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
      TaskState& st = ts[t];
      if (step < a.tasks[t].n_steps && (st.live || st.fail_step == step)) st.it_total += st.it_step;
      st.order = st.order < kCoopOrder ? st.order + 1 : kCoopOrder;
    }
    bool want_energy = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      if (t < 0) continue;
      const mlmcp_task& tk = a.tasks[t];
      const int i = sl.row[r];
      const int64_t o = (int64_t)t * a.N + i;
      if (ts[t].live && step < tk.n_steps) {
        a.ring[(int64_t)(step & (kCoopOrder - 1)) * TN + o] = *xrow(a, a.Xb, t, i);  // a_n joins the ring
        if (tk.traj >= 0) a.xbuf[tk.traj + (int64_t)(step + 1) * a.N + i] = sl.x[r];
      }
    }
    for (int t = 0; t < a.T; ++t)
      want_energy |= ts[t].live && a.tasks[t].qoi_mode == MLMCP_QOI_SUM_ENERGY &&
                     step < a.tasks[t].n_steps && a.tasks[t].k0 + step + 1 > a.tasks[t].qoi_from;
    if (want_energy) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (sl.task[r] >= 0) *xrow(a, a.Xb, sl.task[r], sl.row[r]) = sl.x[r];
      grid_barrier(gb);
      double lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = sl.task[r];
        if (t < 0 || !ts[t].live) continue;
        (t == t_lo ? lo : hi)[0] += sl.x[r] * csr_apply(a, sl, r, a.K, a.Xb);
      }
      cta_partials<4>(lo, hi, t_lo, t_hi, a, red);
      grid_barrier(gb);
      task_totals<1>(a, tot);
      if (blockIdx.x == 0)
        for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
          const mlmcp_task& tk = a.tasks[t];
          if (ts[t].live && tk.qoi_mode == MLMCP_QOI_SUM_ENERGY && tk.qoi_slot >= 0 &&
              step < tk.n_steps && tk.k0 + step + 1 > tk.qoi_from)
            a.qoi[tk.qoi_slot] += 0.5 * tot[t * 4 + 0];   // qoi zeroed by the caller
        }
    }
      }
  // ---- outputs
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int t = sl.task[r];
    if (t < 0) continue;
    const mlmcp_task& tk = a.tasks[t];
    const bool inactive = a.active != nullptr && tk.group >= 0 && a.active[tk.group] == 0 &&
                          ts[t].code == MLMCP_ST_OK;
    if (tk.x_out >= 0 && !inactive) a.xbuf[tk.x_out + sl.row[r]] = sl.x[r];
    *xrow(a, a.Xb, t, sl.row[r]) = sl.x[r];
  }
  bool want_final = false;
  for (int t = 0; t < a.T; ++t)
    want_final |= ts[t].live && a.tasks[t].qoi_mode == MLMCP_QOI_FINAL_ENERGY && a.tasks[t].qoi_slot >= 0;
  if (want_final) {
    grid_barrier(gb);
    double lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = sl.task[r];
      if (t < 0 || !ts[t].live) continue;
      (t == t_lo ? lo : hi)[0] += sl.x[r] * csr_apply(a, sl, r, a.K, a.Xb);
    }
    cta_partials<4>(lo, hi, t_lo, t_hi, a, red);
    grid_barrier(gb);
    task_totals<1>(a, tot);
    if (blockIdx.x == 0)
      for (int t = threadIdx.x; t < a.T; t += kCoopThreads)
        if (ts[t].live && a.tasks[t].qoi_mode == MLMCP_QOI_FINAL_ENERGY && a.tasks[t].qoi_slot >= 0)
          a.qoi[a.tasks[t].qoi_slot] = 0.5 * tot[t * 4 + 0];
  }
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < a.T; t += kCoopThreads) {
      const mlmcp_task& tk = a.tasks[t];
      const TaskState& st = ts[t];
      if (a.iters != nullptr && tk.slot >= 0) a.iters[tk.slot] = st.it_total;
      if (st.code != MLMCP_ST_OK) {
        write_status(a.status, tk.slot, st.code, st.fail_step, tk.tag, tk.tag);
        if (a.active != nullptr && tk.group >= 0) a.active[tk.group] = 0;
      }
    }
  }
}

}  // namespace
}  // namespace mlmcp

namespace mlmcp {
namespace {

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int coop_rows_per_thread(int N) {
  if (N >= 8 * kCoopThreads) return 8;
  // (the stencil-slot operator layout is required: see coop_usable)
  if (N >= 4 * kCoopThreads) return 4;
  return 0;  // too small for this path (rows of > 2 tasks per CTA)
}

struct CoopPlan {
  int R = 0, grid = 0, chunk = 0;
  size_t bytes = 0;
};

CoopPlan coop_plan(const Ctx* ctx, int n_tasks) {
  CoopPlan p;
  p.R = coop_rows_per_thread(ctx->n);
  if (p.R == 0) return p;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.grid = sms;
  const long cap = (long)sms * kCoopThreads * p.R;
  p.chunk = (int)std::min<long>(n_tasks, cap / ctx->n);
  if (p.chunk < 1) { p.R = 0; return p; }
  const size_t TN = (size_t)p.chunk * ctx->n;
  const size_t TL = (size_t)p.chunk * (ctx->n + 2 * ctx->stencil_pad);
  const int nb_task = ctx->n / (kCoopThreads * p.R) + 2;
  p.bytes = al256(3 * TL * 8) + al256(kCoopOrder * TN * 8) +
            al256((size_t)p.chunk * nb_task * 4 * 8) + al256((size_t)p.chunk * 2 * 4);
  return p;
}

template <int R, int W>
int launch_coop(CoopArgs& a, int grid, cudaStream_t stream) {
  const size_t smem = (64 + 4 * (size_t)a.T) * 8 + sizeof(TaskState) * (size_t)a.T;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(coop_kernel<R, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  MLMCP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_kernel<R, W>,
                                                                 kCoopThreads, smem));
  if (per_sm < 1) {
    set_error("cooperative PCG kernel does not fit one CTA per SM");
    return MLMCP_EINVAL;
  }
  void* args[] = {&a};
  MLMCP_CUDA_CHECK(cudaLaunchCooperativeKernel((void*)coop_kernel<R, W>, dim3(grid),
                                               dim3(kCoopThreads), args, smem, stream));
  count_launch();
  return MLMCP_OK;
}

}  // namespace

size_t coop_workspace_bytes(const Ctx* ctx, int n_tasks) { return coop_plan(ctx, n_tasks).bytes; }

bool coop_usable(const Ctx* ctx, int n_tasks) {
  // MLMCP_STREAM_IMPL: 1 two-launch kernels, 2 cooperative, 4 tile, default auto
  const char* e = getenv("MLMCP_STREAM_IMPL");
  const int impl = e ? atoi(e) : 0;
  if (impl == 1 || impl == 4 || ctx->stencil_w == 0) return false;
  const CoopPlan p = coop_plan(ctx, n_tasks);
  if (p.R == 0) return false;
  // auto: the grid-resident kernel is barrier-latency bound (~16 us per PCG
  // iteration); it wins when the whole batch fits one register-resident chunk.
  // Larger batches amortise better in the two-launch streaming kernels.
  return impl == 2 || p.chunk >= n_tasks;
}

int coop_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks_d,
                   const std::vector<mlmcp_task>& h, int S, const double* A,
                   const double* dinv, const double* M, const double* K,
                   const double* profile, double omega, double rtol, int max_it, double* xbuf,
                   double* qoi, int32_t* iters, int32_t* status, const int32_t* active,
                   char* ws, size_t ws_bytes, cudaStream_t stream) {
  const CoopPlan plan = coop_plan(ctx, n_tasks);
  if (plan.R == 0) {
    set_error("cooperative path not applicable");
    return MLMCP_EINVAL;
  }
  if (ws_bytes < plan.bytes) {
    set_error("cooperative workspace too small");
    return MLMCP_ENOMEM;
  }
  const int N = ctx->n;
  const int nb_task = N / (kCoopThreads * plan.R) + 2;
  for (int c0 = 0; c0 < n_tasks; c0 += plan.chunk) {
    const int T = std::min(plan.chunk, n_tasks - c0);
    const size_t TN = (size_t)T * N;
    const int pad = ctx->stencil_pad;
    const size_t TL = (size_t)T * (N + 2 * pad);
    char* b = ws;
    CoopArgs a{};
    a.Xb = reinterpret_cast<double*>(b);
    a.Gb = a.Xb + TL;
    a.Ub = a.Gb + TL;
    MLMCP_CUDA_CHECK(cudaMemsetAsync(a.Xb, 0, 3 * TL * 8, stream));   // zero pads
    MLMCP_CUDA_CHECK(cudaMemsetAsync(ctx->grid_bar, 0, (1 + 1024) * sizeof(unsigned int), stream));
    b += al256(3 * TL * 8);
    a.ring = reinterpret_cast<double*>(b);
    b += al256(kCoopOrder * TN * 8);
    a.part = reinterpret_cast<double*>(b);
    b += al256((size_t)T * nb_task * 4 * 8);
    int32_t* blk = reinterpret_cast<int32_t*>(b);
    std::vector<int32_t> hb(2 * T);
    const long rows_per_cta = (long)kCoopThreads * plan.R;
    for (int t = 0; t < T; ++t) {
      const long f = (long)t * N / rows_per_cta, l = ((long)(t + 1) * N - 1) / rows_per_cta;
      hb[t] = (int32_t)f;
      hb[T + t] = (int32_t)(l - f + 1);
    }
    MLMCP_CUDA_CHECK(cudaMemcpyAsync(blk, hb.data(), sizeof(int32_t) * 2 * T,
                                     cudaMemcpyHostToDevice, stream));
    a.first_blk = blk;
    a.n_blk = blk + T;
    a.T = T;
    a.N = N;
    a.R = plan.R;
    a.S = S;
    a.nb_task = nb_task;
    a.pad = pad;
    a.ld = N + 2 * pad;
    a.bar = ctx->grid_bar;
    a.epoch0 = 0;
    for (int k = 0; k < kMaxNz; ++k) a.off[k] = k < ctx->stencil_w ? ctx->stencil_off[k] : 0;
    a.W = ctx->stencil_w;
    a.tasks = tasks_d + c0;
    a.A = A;
    a.dinv = dinv;
    a.ell_col = ctx->ell_col;
    a.row_ptr = ctx->row_ptr;
    a.col = ctx->col;
    a.M = M;
    a.K = K;
    a.nnz = ctx->nnz;
    a.profile = profile;
    a.omega = omega;
    a.rtol2 = rtol * rtol;
    a.max_it = max_it;
    a.xbuf = xbuf;
    a.qoi = qoi;
    a.iters = iters;
    a.status = status;
    a.active = const_cast<int32_t*>(active);
    int rc = MLMCP_EINVAL;
    set_error("unsupported stencil width for the cooperative path");
#define MLMCP_COOP_W(WW)                                                              \
    if (a.W == WW)                                                                    \
      rc = plan.R == 8 ? launch_coop<8, WW>(a, plan.grid, stream)                     \
                       : launch_coop<4, WW>(a, plan.grid, stream);
    MLMCP_COOP_W(3) MLMCP_COOP_W(5) MLMCP_COOP_W(7)
#undef MLMCP_COOP_W
    if (rc != MLMCP_OK) return rc;
    // the host vector hb must outlive the async copy: synchronise the copy
    MLMCP_CUDA_CHECK(cudaStreamSynchronize(stream));
  }
  (void)h;
  return MLMCP_OK;
}

}  // namespace mlmcp
