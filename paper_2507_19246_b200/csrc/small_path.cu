// small_path.cu — SM-resident batched implicit Euler (one CTA per task).
//
// Replaces the per-step dense LU solve of the reference
// (timeint.py:64-75 factorise, :108-110 / :126-127 per-step solve) for
// meshes whose interior system has <= 1024 rows (the 32x32 mesh of configs
// 0/1 has 961).  Each CTA (256 threads) owns one (sample, slice) task for its
// lifetime; a thread owns 4 rows, whose <= 8 coefficients of A = M + dt*K and
// D^-1 sit in registers for every step and every PCG iteration (no HBM
// traffic for the operator after the first load).
//
// The SpMV operand exchange is an "operator" policy (publish -> barrier ->
// apply):
//   GridOp     structured 7-point FE stencil on a wd x h <= 32 x 32 grid:
//              thread (warp w, lane l) owns grid points (x=l, y=4w+k); N/S
//              neighbours come from the thread's own registers, E/W (and
//              NE/SW) from warp shuffles, only the warp-tile halos (2 values
//              per lane) go through shared memory.
//   StencilOp  uniform-offset stencil (every col-row in <= 8 offsets): rows
//              tid + 256k, neighbour j read from a zero-padded smem vector at
//              a block-uniform offset.
//   CsrOp      generic pattern: packed 16-bit smem byte offsets per entry.
// PCG is the Chronopoulos-Gear single-reduction variant: one fused block
// all-reduce (r.u, w.u, r.r) per iteration, two __syncthreads; the alpha/beta
// recurrence has one reciprocal on the critical path.  The cross-warp stage
// of the reduction is a broadcast smem read of the 8 warp partials + a fixed
// tree, so every thread holds bitwise identical totals (deterministic).
// The QoI (magnetic energy 1/2 x^T K x) is fused into the step loop.
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
constexpr int kHaloLd = 34;                       // grid halo row: 32 lanes + 2 pads
constexpr int kHaloRows = kMaxWarps + 2;          // 8 warps + 2 zero rows
constexpr int kHaloBuf = 2 * kHaloRows * kHaloLd; // lo + hi halos

struct PatternArgs {
  int N;
  const int32_t* row_ptr;
  const int32_t* col;
  int off[kMaxNz];       // stencil: sorted offsets (col - row)
  int off8[kMaxNz];      // the same in bytes
  const int32_t* spos;   // stencil: [W][N] CSR position of slot j of row i, or -1
  int pad;               // stencil: zero rows before row 0 / after the last padded row
  int wd, gh;            // grid: width / height
  const int32_t* gpos;   // grid: [7][N] CSR position per direction, or -1
};

__device__ __forceinline__ double lds_off(const double* base, uint32_t off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + off);
}

// ---------------------------------------------------------------- block reduce
// Block all-reduce of NV <= 4 doubles.  Butterfly inside each warp, then every
// thread reads the 8 warp partials (broadcast) and sums them in a fixed tree.
template <int NV>
__device__ __forceinline__ void cta_allsum(double (&v)[NV], double* red, int& par) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  double* buf = red + par * (kMaxWarps * 4);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) buf[warp * 4 + k] = v[k];
  }
  __syncthreads();
  auto ld = [&](int w, double (&o)[NV]) {
    const double2 lo = *reinterpret_cast<const double2*>(buf + w * 4);
    o[0] = lo.x;
    if (NV > 1) o[1 % NV] = lo.y;
    if (NV > 2) {
      const double2 hi = *reinterpret_cast<const double2*>(buf + w * 4 + 2);
      o[2 % NV] = hi.x;
      if (NV > 3) o[3 % NV] = hi.y;
    }
  };
  static_assert(kMaxWarps == 8, "tree below is written for 8 warps");
  // fixed tree ((w0+w1)+(w2+w3))+((w4+w5)+(w6+w7)), streamed (few live regs)
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
  par ^= 1;
}

// ---------------------------------------------------------------- operators
// Common interface (R = rows per thread):
//   load(pa, Ms, Ks, dt)               coefficients of A = M + dt K, D^-1
//   ok(r, pa), row(r, pa)              validity / global row of slot r
//   publish(v, buf, pa)                store what neighbours need (before a barrier)
//   apply(v, buf, pa, out)             out = A v (register coefficients)
//   apply_vals(vals, v, buf, pa, out)  out = B v (B: per-sample CSR values)
//   buffer_doubles(pad)                smem doubles of one exchange buffer
// Invalid (padding) slots hold v = 0, a = 0, dinv = 0.

template <int W, int R_>
struct StencilOp {
  static constexpr int R = R_;
  double a[R][W];
  double dinv[R];
  __device__ static int row(int r, const PatternArgs&) { return threadIdx.x + r * kSmallThreads; }
  __device__ static bool ok(int r, const PatternArgs& pa) { return row(r, pa) < pa.N; }
  static int buffer_doubles(int pad) { return pad + R * kSmallThreads + pad; }

  __device__ void load(const PatternArgs& pa, const double* __restrict__ Ms,
                       const double* __restrict__ Ks, double dt) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool v = ok(r, pa);
      double diag = 1.0;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int q = v ? pa.spos[j * pa.N + row(r, pa)] : -1;
        a[r][j] = q >= 0 ? op_entry(__ldg(Ms + q), __ldg(Ks + q), dt) : 0.0;
        if (pa.off[j] == 0 && q >= 0) diag = a[r][j];
      }
      dinv[r] = v ? 1.0 / diag : 0.0;
    }
  }
  __device__ static double* base(double* buf, const PatternArgs& pa) { return buf + pa.pad; }
  __device__ void publish(const double (&v)[R], double* buf, const PatternArgs& pa) const {
#pragma unroll
    for (int r = 0; r < R; ++r) base(buf, pa)[row(r, pa)] = v[r];  // padded: every slot writes
  }
  __device__ void apply(const double (&v)[R], double* buf, const PatternArgs& pa,
                        double (&out)[R]) const {
    const double* b = base(buf, pa);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        acc0 = fma(a[r][j], lds_off(b + row(r, pa), (uint32_t)pa.off8[j]), acc0);
        if (j + 1 < W)
          acc1 = fma(a[r][j + 1], lds_off(b + row(r, pa), (uint32_t)pa.off8[j + 1]), acc1);
      }
      out[r] = acc0 + acc1;
    }
  }
  __device__ void apply_vals(const double* __restrict__ vals, const double (&v)[R], double* buf,
                             const PatternArgs& pa, double (&out)[R]) const {
    const double* b = base(buf, pa);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if (ok(r, pa)) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int q = __ldg(pa.spos + j * pa.N + row(r, pa));
          if (q >= 0) acc = fma(__ldg(vals + q), b[row(r, pa) + pa.off[j]], acc);
        }
      }
      out[r] = acc;
    }
  }
};

template <int W, int R_>
struct CsrOp {
  static constexpr int R = R_;
  double a[R][W];
  uint32_t cp[R][(W + 1) / 2];  // packed 16-bit smem byte offsets of the columns
  double dinv[R];
  __device__ static int row(int r, const PatternArgs&) { return threadIdx.x + r * kSmallThreads; }
  __device__ static bool ok(int r, const PatternArgs& pa) { return row(r, pa) < pa.N; }
  static int buffer_doubles(int) { return R * kSmallThreads; }
  __device__ uint32_t off(int r, int j) const {
    const uint32_t w = cp[r][j >> 1];
    return (j & 1) ? (w >> 16) : (w & 0xffffu);
  }

  __device__ void load(const PatternArgs& pa, const double* __restrict__ Ms,
                       const double* __restrict__ Ks, double dt) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int rw = row(r, pa);
      const bool v = ok(r, pa);
      const int q0 = v ? pa.row_ptr[rw] : 0;
      const int len = v ? pa.row_ptr[rw + 1] - q0 : 0;
      double diag = 1.0;
#pragma unroll
      for (int j = 0; j < (W + 1) / 2; ++j) cp[r][j] = 0u;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        uint32_t o;
        if (j < len) {
          const int q = q0 + j;
          const int c = pa.col[q];
          o = (uint32_t)c * 8u;
          a[r][j] = op_entry(__ldg(Ms + q), __ldg(Ks + q), dt);
          if (c == rw) diag = a[r][j];
        } else {
          o = v ? (uint32_t)rw * 8u : 0u;
          a[r][j] = 0.0;
        }
        cp[r][j >> 1] |= (j & 1) ? (o << 16) : o;
      }
      dinv[r] = v ? 1.0 / diag : 0.0;
    }
  }
  __device__ void publish(const double (&v)[R], double* buf, const PatternArgs& pa) const {
#pragma unroll
    for (int r = 0; r < R; ++r) buf[row(r, pa)] = v[r];
  }
  __device__ void apply(const double (&v)[R], double* buf, const PatternArgs&,
                        double (&out)[R]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        acc0 = fma(a[r][j], lds_off(buf, off(r, j)), acc0);
        if (j + 1 < W) acc1 = fma(a[r][j + 1], lds_off(buf, off(r, j + 1)), acc1);
      }
      out[r] = acc0 + acc1;
    }
  }
  __device__ void apply_vals(const double* __restrict__ vals, const double (&v)[R], double* buf,
                             const PatternArgs& pa, double (&out)[R]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if (ok(r, pa)) {
        const int q0 = __ldg(pa.row_ptr + row(r, pa));
        const int len = __ldg(pa.row_ptr + row(r, pa) + 1) - q0;
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (j < len) acc = fma(__ldg(vals + q0 + j), lds_off(buf, off(r, j)), acc);
      }
      out[r] = acc;
    }
  }
};

// Structured 7-point stencil, directions SW,S,W,C,E,N,NE = slots 0..6.
struct GridOp {
  static constexpr int R = 4;
  double a[R][7];
  double dinv[R];
  __device__ static int lane() { return threadIdx.x & 31; }
  __device__ static int warp() { return threadIdx.x >> 5; }
  __device__ static int gy(int r) { return 4 * warp() + r; }
  __device__ static bool ok(int r, const PatternArgs& pa) { return lane() < pa.wd && gy(r) < pa.gh; }
  __device__ static int row(int r, const PatternArgs& pa) { return gy(r) * pa.wd + lane(); }
  static int buffer_doubles(int) { return kHaloBuf; }

  __device__ void load(const PatternArgs& pa, const double* __restrict__ Ms,
                       const double* __restrict__ Ks, double dt) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool v = ok(r, pa);
      const int rw = v ? row(r, pa) : 0;
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        const int q = v ? pa.gpos[j * pa.N + rw] : -1;
        a[r][j] = q >= 0 ? op_entry(__ldg(Ms + q), __ldg(Ks + q), dt) : 0.0;
      }
      dinv[r] = (v && a[r][3] != 0.0) ? 1.0 / a[r][3] : 0.0;
    }
  }
  // halo rows: lo[w+1][l+1] = v[0] of warp w, hi[w+1][l+1] = v[3]
  __device__ void publish(const double (&v)[R], double* buf, const PatternArgs&) const {
    const int i = (warp() + 1) * kHaloLd + lane() + 1;
    buf[i] = v[0];
    buf[kHaloRows * kHaloLd + i] = v[3];
  }
  // the 7 neighbour values of each slot
  __device__ void neighbours(const double (&v)[R], const double* buf, double (&nb)[R][7]) const {
    double e[R], w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      e[r] = __shfl_down_sync(0xffffffffu, v[r], 1);
      w[r] = __shfl_up_sync(0xffffffffu, v[r], 1);
    }
    const double* lo = buf;
    const double* hi = buf + kHaloRows * kHaloLd;
    const int up = (warp() + 2) * kHaloLd + lane() + 1;   // warp w+1, lane l
    const int dn = warp() * kHaloLd + lane() + 1;         // warp w-1, lane l
    const double n3 = lo[up], ne3 = lo[up + 1];
    const double s0 = hi[dn], sw0 = hi[dn - 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      nb[r][0] = r > 0 ? w[r - 1] : sw0;
      nb[r][1] = r > 0 ? v[r - 1] : s0;
      nb[r][2] = w[r];
      nb[r][3] = v[r];
      nb[r][4] = e[r];
      nb[r][5] = r < R - 1 ? v[r + 1] : n3;
      nb[r][6] = r < R - 1 ? e[r + 1] : ne3;
    }
  }
  __device__ void apply(const double (&v)[R], double* buf, const PatternArgs&,
                        double (&out)[R]) const {
    double nb[R][7];
    neighbours(v, buf, nb);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc0 = a[r][3] * nb[r][3];
      double acc1 = a[r][0] * nb[r][0];
      acc0 = fma(a[r][1], nb[r][1], acc0);
      acc1 = fma(a[r][2], nb[r][2], acc1);
      acc0 = fma(a[r][4], nb[r][4], acc0);
      acc1 = fma(a[r][5], nb[r][5], acc1);
      acc0 = fma(a[r][6], nb[r][6], acc0);
      out[r] = acc0 + acc1;
    }
  }
  __device__ void apply_vals(const double* __restrict__ vals, const double (&v)[R], double* buf,
                             const PatternArgs& pa, double (&out)[R]) const {
    double nb[R][7];
    neighbours(v, buf, nb);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if (ok(r, pa)) {
        const int rw = row(r, pa);
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          const int q = __ldg(pa.gpos + j * pa.N + rw);
          if (q >= 0) acc = fma(__ldg(vals + q), nb[r][j], acc);
        }
      }
      out[r] = acc;
    }
  }
};

struct SmallShared {
  double* bufA;  // exchange buffer for a_n (M a_n) and the energy
  double* bufB;  // exchange buffer for the initial guess (A x0)
  double* bufC;  // exchange buffer for u (PCG iterations)
  double* red;   // [2][kMaxWarps][4]
  double* ring;  // [kMaxOrder][R*256] state history (per-thread slots)
  int par;
};

// State history of the current task for the PCG initial guess: the guess is
// the polynomial extrapolation of the last p+1 states,
//     x0 = sum_{i=0..p} (-1)^i C(p+1, i+1) a_{n-i},   p = min(#history, kMaxOrder),
// (p = 0: a_n; 1: 2a_n - a_{n-1}; 2: 3a_n - 3a_{n-1} + a_{n-2}; ...).  Only the
// starting point of PCG changes — the stopping rule ||r|| <= rtol ||b|| and
// hence the accuracy of every step are unchanged — but the initial residual
// drops by ~O(omega dt) per order (configs 0/1: 59 -> 26 PCG iterations per
// step at T/256, 51 -> 16 at T/1024 for p = 4).  The past states live in a
// per-thread shared-memory ring (touched once per step), a_n in registers.
constexpr int kMaxOrder = 4;

template <int R>
struct StateHistory {
  double* ring;   // [kMaxOrder][R*256]: a_{n-1} .. a_{n-4} (ring)
  int head;       // ring slot of a_{n-1}
  int count;      // valid past states (<= kMaxOrder)
  int max_order;  // 0 disables extrapolation (MLMCP_TASK_NO_EXTRAPOLATION)
  __device__ StateHistory(double* ring_, int max_ord)
      : ring(ring_), head(kMaxOrder - 1), count(0), max_order(max_ord) {}
  __device__ double past(int i, int r) const {  // a_{n-i}, i >= 1
    const int slot = (head - (i - 1) + kMaxOrder) % kMaxOrder;
    return ring[slot * (R * kSmallThreads) + r * kSmallThreads + threadIdx.x];
  }
  // on entry x = a_n; on exit x = initial guess, an = a_n; a_n joins the ring
  __device__ void advance(double (&x)[R], double (&an)[R]) {
    const int p = count < max_order ? count : max_order;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      an[r] = x[r];
      double g;
      switch (p) {
        case 0: g = an[r]; break;
        case 1: g = fma(2.0, an[r], -past(1, r)); break;
        case 2: g = fma(3.0, an[r] - past(1, r), past(2, r)); break;
        case 3: g = fma(4.0, an[r] + past(2, r), fma(-6.0, past(1, r), -past(3, r))); break;
        default:  // 5a_n - 10a_{n-1} + 10a_{n-2} - 5a_{n-3} + a_{n-4}
          g = fma(5.0, an[r] - past(3, r), fma(10.0, past(2, r) - past(1, r), past(4, r)));
          break;
      }
      x[r] = g;
    }
    head = (head + 1) % kMaxOrder;
#pragma unroll
    for (int r = 0; r < R; ++r)
      ring[head * (R * kSmallThreads) + r * kSmallThreads + threadIdx.x] = an[r];
    count = count < kMaxOrder ? count + 1 : kMaxOrder;
  }
};

// 1/2 x^T K x over the block (every thread receives it).  Uses bufA.
template <class Op>
__device__ __forceinline__ double block_energy(const Op& op, const double (&x)[Op::R],
                                               const PatternArgs& pa,
                                               const double* __restrict__ Ks, SmallShared& sh) {
  constexpr int R = Op::R;
  op.publish(x, sh.bufA, pa);
  __syncthreads();
  double kx[R];
  op.apply_vals(Ks, x, sh.bufA, pa, kx);
  double v[1] = {0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) v[0] = fma(x[r], kx[r], v[0]);
  cta_allsum<1>(v, sh.red, sh.par);
  return 0.5 * v[0];
}

// One implicit-Euler step (M + dt K) a_{n+1} = M a_n + dt*sf*profile by
// Chronopoulos-Gear Jacobi-PCG.  x holds the initial guess on entry (the
// caller extrapolates it from the state history) and a_{n+1} on exit.
// Returns MLMCP_ST_*.
template <class Op>
__device__ __forceinline__ int ie_step(const Op& op, double (&x)[Op::R], const double (&an)[Op::R],
                                       const PatternArgs& pa, double sf, double dt,
                                       const double* __restrict__ Ms,
                                       const double* __restrict__ profile, double rtol2,
                                       int max_it, SmallShared& sh, int& iters) {
  constexpr int R = Op::R;
  // b = M a_n + dt*(sf*prof);  r = b - A x0;  u = D r;  w = A u
  op.publish(an, sh.bufA, pa);
  op.publish(x, sh.bufB, pa);
  __syncthreads();
  double res[R], u[R], p[R], s[R], w[R], mx[R], ax[R];
  op.apply_vals(Ms, an, sh.bufA, pa, mx);
  op.apply(x, sh.bufB, pa, ax);
  double red4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    res[r] = 0.0;
    u[r] = 0.0;
    if (Op::ok(r, pa)) {
      const int rw = Op::row(r, pa);
      const double b = __dadd_rn(mx[r], __dmul_rn(dt, __dmul_rn(sf, __ldg(profile + rw))));
      res[r] = b - ax[r];
      u[r] = op.dinv[r] * res[r];
      red4[3] += b * b;
    }
  }
  op.publish(u, sh.bufC, pa);
  __syncthreads();
  op.apply(u, sh.bufC, pa, w);                    // a = 0 on padding slots
#pragma unroll
  for (int r = 0; r < R; ++r) {
    red4[0] += res[r] * u[r];
    red4[1] += w[r] * u[r];
    red4[2] += res[r] * res[r];
  }
  cta_allsum<4>(red4, sh.red, sh.par);
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
    for (int r = 0; r < R; ++r) u[r] = op.dinv[r] * res[r];   // 0 on padding slots
    op.publish(u, sh.bufC, pa);
    __syncthreads();
    op.apply(u, sh.bufC, pa, w);
    double red3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      red3[0] = fma(res[r], u[r], red3[0]);
      red3[1] = fma(w[r], u[r], red3[1]);
      red3[2] = fma(res[r], res[r], red3[2]);
    }
    cta_allsum<3>(red3, sh.red, sh.par);
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
    alpha = gnew * fast_rcp(den);
    inv_g = fast_rcp(gnew);                // off the critical path (next iteration)
    c = inv_g * (den * inv_g);             // 1/(gnew*alpha)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      p[r] = fma(beta, p[r], op.dinv[r] * res[r]);   // u recomputed: fewer live registers
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
  int64_t nnz;
  PatternArgs pa;
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
  int64_t* elapsed;
  int buf_doubles;
};

// Carve and zero the exchange buffers.
__device__ __forceinline__ SmallShared setup_shared(double* smem, int len) {
  for (int i = threadIdx.x; i < 3 * len; i += kSmallThreads) smem[i] = 0.0;
  __syncthreads();
  return SmallShared{smem, smem + len, smem + 2 * len, smem + 3 * len,
                     smem + 3 * len + 2 * kMaxWarps * 4, 0};
}

template <class Op, int OCC>
__global__ void __launch_bounds__(kSmallThreads, OCC) small_propagate_kernel(SmallArgs a) {
  constexpr int R = Op::R;
  extern __shared__ __align__(16) double smem[];
  const mlmcp_task t = a.tasks[blockIdx.x];
  const int64_t t_start = global_ns();
  {
    // another CTA of the same group may clear active[] concurrently (on a
    // failure): decide once per block so the barriers below never diverge
    __shared__ int skip;
    if (threadIdx.x == 0)
      skip = (a.active != nullptr && t.group >= 0 && a.active[t.group] == 0) ? 1 : 0;
    __syncthreads();
    if (skip) return;
  }
  const PatternArgs& pa = a.pa;
  SmallShared sh = setup_shared(smem, a.buf_doubles);
  const double* Ms = a.M + (int64_t)t.sample * a.nnz;
  const double* Ks = a.K + (int64_t)t.sample * a.nnz;
  Op op;
  op.load(pa, Ms, Ks, t.dt);
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool v = Op::ok(r, pa);
    const int rw = v ? Op::row(r, pa) : 0;
    x[r] = v ? a.xbuf[t.x_in + rw] : 0.0;
    if (t.traj >= 0 && v) a.xbuf[t.traj + rw] = x[r];
  }
  int iters = 0;
  int code = MLMCP_ST_OK;
  int fail_step = 0;
  double acc = 0.0;
  StateHistory<R> hist(sh.ring, (t.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : kMaxOrder);
  double an[R];
  for (int step = 0; step < t.n_steps; ++step) {
    const int64_t g = t.k0 + step + 1;
    const double sf = sin(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)));
    hist.advance(x, an);                   // x <- extrapolated initial guess
    code = ie_step<Op>(op, x, an, pa, sf, t.dt, Ms, a.profile, a.rtol2, a.max_it, sh, iters);
    if (code != MLMCP_ST_OK) { fail_step = step; break; }
    if (t.traj >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (Op::ok(r, pa)) a.xbuf[t.traj + (int64_t)(step + 1) * pa.N + Op::row(r, pa)] = x[r];
    }
    if (g > t.qoi_from) {
      if (t.qoi_mode == MLMCP_QOI_SUM_ENERGY) {
        acc += block_energy<Op>(op, x, pa, Ks, sh);
      } else if (t.qoi_mode == MLMCP_QOI_JOULE) {
        double d[R];
#pragma unroll
        for (int r = 0; r < R; ++r) d[r] = x[r] - an[r];   // 0 on padding slots
        acc += 2.0 * block_energy<Op>(op, d, pa, Ms, sh);
      } else if (t.qoi_mode == MLMCP_QOI_ELECTRICAL) {
#pragma unroll
        for (int r = 0; r < R; ++r)   // only the owner of row qoi_index accumulates
          if (Op::ok(r, pa) && Op::row(r, pa) == t.qoi_index)
            acc = __dadd_rn(acc, __dmul_rn(sf, x[r]));
      }
    }
  }
  if (t.x_out >= 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (Op::ok(r, pa)) a.xbuf[t.x_out + Op::row(r, pa)] = x[r];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY && t.qoi_slot >= 0)
    acc = block_energy<Op>(op, x, pa, Ks, sh);
  if (t.qoi_mode == MLMCP_QOI_ELECTRICAL && t.qoi_slot >= 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (Op::ok(r, pa) && Op::row(r, pa) == t.qoi_index) a.qoi[t.qoi_slot] = acc;
  }
  if (threadIdx.x == 0) {
    if (t.qoi_slot >= 0 && t.qoi_mode != MLMCP_QOI_NONE && t.qoi_mode != MLMCP_QOI_ELECTRICAL)
      a.qoi[t.qoi_slot] = acc;
    if (a.iters != nullptr && t.slot >= 0) a.iters[t.slot] = iters;
    add_elapsed(a.elapsed, t.slot, t_start);
    if (code != MLMCP_ST_OK) {
      write_status(a.status, t.slot, code, fail_step, t.tag, t.tag);
      if (a.active != nullptr && t.group >= 0) a.active[t.group] = 0;
    }
  }
}

struct CoarseArgs {
  int S, k, m;
  int64_t nnz;
  PatternArgs pa;
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
  int64_t* elapsed;
  int buf_doubles;
};

// parareal.py:168-178 for one sample per CTA.
template <class Op, int OCC>
__global__ void __launch_bounds__(kSmallThreads, OCC) small_coarse_kernel(CoarseArgs a) {
  constexpr int R = Op::R;
  extern __shared__ __align__(16) double smem[];
  const int s = blockIdx.x;
  const int64_t t_start = global_ns();
  if (a.active[s] == 0) return;
  const PatternArgs& pa = a.pa;
  SmallShared sh = setup_shared(smem, a.buf_doubles);
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  Op op;
  op.load(pa, Ms, Ks, a.dt);
  const int64_t N = pa.N;
  double* U = a.U + (int64_t)s * (a.m + 1) * N;
  const double* F = a.F + (int64_t)s * (a.m + 1) * N;
  double* C = a.C + (int64_t)s * a.m * N;
  int iters = 0;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool v = Op::ok(r, pa);
    const int i = v ? Op::row(r, pa) : 0;
    if (a.k == 1) {
      x[r] = v ? U[i] : 0.0;
    } else {
      x[r] = v ? F[(a.k - 1) * N + i] : 0.0;  // freeze U_{k-1} = F_{k-1}
      if (v) U[(a.k - 1) * N + i] = x[r];
    }
  }
  for (int n = a.k; n < a.m; ++n) {
    const int steps = a.slice_steps[n - 1];
    const int64_t k0 = a.slice_k0[n - 1];
    StateHistory<R> hist(sh.ring, kMaxOrder);
    double an[R];
    for (int step = 0; step < steps; ++step) {
      const int64_t g = k0 + step + 1;
      const double sf = sin(__dmul_rn(a.omega, grid_time(a.t0, g, a.dt)));
      hist.advance(x, an);
      const int code = ie_step<Op>(op, x, an, pa, sf, a.dt, Ms, a.profile, a.rtol2,
                                   a.max_it, sh, iters);
      if (code != MLMCP_ST_OK) {
        if (threadIdx.x == 0) {
          write_status(a.status, s, code, step, n, a.k);
          a.active[s] = 0;
          if (a.iters != nullptr) a.iters[s] += iters;
          add_elapsed(a.elapsed, s, t_start);
        }
        return;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!Op::ok(r, pa)) continue;
      const int i = Op::row(r, pa);
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
    for (int r = 0; r < R; ++r)
      if (Op::ok(r, pa)) {
        const int i = Op::row(r, pa);
        U[a.m * N + i] = F[a.m * N + i];
      }
  }
  if (threadIdx.x == 0) {
    if (a.iters != nullptr) a.iters[s] += iters;
    add_elapsed(a.elapsed, s, t_start);
  }
  (void)Ks;
}

inline int rows_per_thread(int N) {
  if (N <= kSmallThreads) return 1;
  if (N <= 2 * kSmallThreads) return 2;
  return 4;
}
inline size_t small_smem(int buf_doubles, int R) {
  return (size_t)(3 * buf_doubles + 2 * kMaxWarps * 4 + kMaxOrder * R * kSmallThreads) *
         sizeof(double);
}

// kernel variant: 0 auto (grid > stencil > csr), 1 no grid tiling (tests / A-B)
int variant_pref() {
  static const int v = [] {
    const char* e = getenv("MLMCP_SMALL_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}
// CTAs per SM for the grid-tiled kernel: 2 (128 registers, two independent
// samples hide each other's reduction latency; measured -10% time on config 1)
// unless MLMCP_SMALL_OCC=1.
int occ_pref() {
  static const int o = [] {
    const char* e = getenv("MLMCP_SMALL_OCC");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return o;
}

template <template <class, int> class Launch, typename Args>
int dispatch(const Ctx* ctx, Args& a, unsigned grid, cudaStream_t stream) {
  const int N = ctx->n;
  PatternArgs& pa = a.pa;
  pa.N = N;
  pa.row_ptr = ctx->row_ptr;
  pa.col = ctx->col;
  pa.pad = 0;
  pa.spos = nullptr;
  pa.gpos = nullptr;
  pa.wd = pa.gh = 0;
  const int occ = occ_pref();
  if (ctx->grid_wd > 0 && variant_pref() != 1) {
    pa.wd = ctx->grid_wd;
    pa.gh = ctx->grid_h;
    pa.gpos = ctx->grid_pos;
    a.buf_doubles = GridOp::buffer_doubles(0);
    const size_t smem = small_smem(a.buf_doubles, GridOp::R);
    return occ == 2 ? Launch<GridOp, 2>::run(a, grid, kSmallThreads, smem, stream)
                    : Launch<GridOp, 1>::run(a, grid, kSmallThreads, smem, stream);
  }
  const int R = rows_per_thread(N);
  const bool st = ctx->stencil_w > 0;
  const int W = st ? ctx->stencil_w : ctx->max_row_nnz;
  if (st) {
    pa.pad = ctx->stencil_pad;
    pa.spos = ctx->stencil_pos;
    for (int k = 0; k < kMaxNz; ++k) {
      pa.off[k] = k < W ? ctx->stencil_off[k] : 0;
      pa.off8[k] = pa.off[k] * 8;
    }
  }
  a.buf_doubles = R * kSmallThreads + 2 * pa.pad;
  const size_t smem = small_smem(a.buf_doubles, R);
  if (smem > 200 * 1024) {
    set_error("SM-resident path: shared-memory footprint too large for this pattern");
    return MLMCP_EINVAL;
  }
#define MLMCP_CASE_R(WW, RR)                                                              \
  if (W == WW && R == RR)                                                                 \
    return st ? Launch<StencilOp<WW, RR>, 1>::run(a, grid, kSmallThreads, smem, stream)   \
              : Launch<CsrOp<WW, RR>, 1>::run(a, grid, kSmallThreads, smem, stream);
#define MLMCP_CASE(WW) MLMCP_CASE_R(WW, 1) MLMCP_CASE_R(WW, 2) MLMCP_CASE_R(WW, 4)
  MLMCP_CASE(1) MLMCP_CASE(2) MLMCP_CASE(3) MLMCP_CASE(4)
  MLMCP_CASE(5) MLMCP_CASE(6) MLMCP_CASE(7) MLMCP_CASE(8)
#undef MLMCP_CASE
#undef MLMCP_CASE_R
  set_error("unsupported row width");
  return MLMCP_EINVAL;
}

template <class Op, int OCC>
struct LaunchPropagate {
  static int run(const SmallArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(small_propagate_kernel<Op, OCC>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    small_propagate_kernel<Op, OCC><<<grid, nt, smem, st>>>(a);
    MLMCP_LAUNCH_CHECK("small_propagate_kernel");
    return MLMCP_OK;
  }
};

template <class Op, int OCC>
struct LaunchCoarse {
  static int run(const CoarseArgs& a, unsigned grid, int nt, size_t smem, cudaStream_t st) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(small_coarse_kernel<Op, OCC>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    small_coarse_kernel<Op, OCC><<<grid, nt, smem, st>>>(a);
    MLMCP_LAUNCH_CHECK("small_coarse_kernel");
    return MLMCP_OK;
  }
};

}  // namespace

int small_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* M,
                    const double* K, const double* profile, double omega, double rtol,
                    int max_it, double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                    const int32_t* active, int64_t* elapsed, cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  SmallArgs a{};
  a.elapsed = elapsed;
  a.tasks = tasks;
  a.n_tasks = n_tasks;
  a.nnz = ctx->nnz;
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
                          int32_t* status, const int32_t* active, int64_t* elapsed,
                          cudaStream_t stream) {
  if (S == 0) return MLMCP_OK;
  CoarseArgs a{};
  a.elapsed = elapsed;
  a.S = S;
  a.k = k;
  a.m = m;
  a.nnz = ctx->nnz;
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
