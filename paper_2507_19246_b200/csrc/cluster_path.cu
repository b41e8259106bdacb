// cluster_path.cu — SM-resident implicit Euler for structured meshes that do
// not fit one SM but fit one thread-block cluster (the 128^2 mesh of config 3:
// 16,129 unknowns).
//
// Same numerical method and step semantics as small_path.cu (reference:
// timeint.py:88-128; every step a Chronopoulos-Gear PCG solve with the
// Jacobi-weighted stopping rule r.D^-1.r <= rtol^2 b.D^-1.b, 4-row strip
// block-Jacobi, extrapolated initial guess), but one task runs on a CLUSTER of
// CS CTAs, one per SM:
//   * CTA c of the cluster owns the band of grid rows [c*HB, (c+1)*HB) of the
//     wd x gh interior grid; each thread a column strip of R rows;
//   * A = M + dt K (7 coefficients per row, the S one implied by symmetry) and
//     the strip's L D L^T factors stay in registers for the whole task; the
//     per-step rhs M a_n reads the per-sample CSR mass values (L2), which
//     leaves shared memory for a ring of 8 past states (order-7 extrapolated
//     initial guesses);
//   * neighbour values go through a shared-memory exchange buffer; a band's
//     first and last grid rows are also stored straight into the neighbouring
//     CTAs' buffers (DSMEM), made visible by one cluster barrier;
//   * the two PCG dot products: warp butterfly, each warp's totals stored into
//     every CTA of the cluster, one cluster barrier, then every CTA sums the
//     CS x warps partials in the same fixed order — bitwise identical scalars
//     in all CTAs, hence one control flow for the whole cluster.
// A PCG iteration touches no global memory.  The HBM-streaming path moves
// B_it = 8 nnz + 56 N bytes (1.8 MB at 128^2) per iteration and task.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

namespace cg = cooperative_groups;

struct ClArgs {
  const mlmcp_task* tasks;
  int N, wd, gh;
  int64_t nnz;
  const int32_t* gpos;   // [7][N]: CSR position of direction SW,S,W,C,E,N,NE, or -1
  const double* M;
  const double* K;
  const double* M7;      // [S][7][N] mass values in stencil-slot layout (direct loads), or null
  int dbg_sync;          // MLMCP_CLUSTER_SYNC=1 (race check of the mbarrier protocol)
  const double* profile;
  double omega, rtol2;
  int max_it;
  int order;             // extrapolation order of the initial guess (<= kRing)
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  const int32_t* active;
  int64_t* elapsed;
};

// R rows per thread strip, TX column threads, NS strips per CTA, CS CTAs per
// cluster: a cluster covers a TX x (CS * R * NS) grid.
template <int R_, int TX_, int NS_, int CS_>
struct Cfg {
  static constexpr int R = R_, TX = TX_, NS = NS_, CS = CS_;
  static constexpr int kThreads = TX * NS;
  static constexpr int kWarps = kThreads / 32;
  static constexpr int HB = R * NS;              // grid rows per CTA
  static constexpr int LD = TX + 2;              // exchange-buffer row stride
  static constexpr int kV = (HB + 2) * LD;       // one exchange buffer (+ halo rows, pad columns)
  static constexpr int kSlots = HB * TX;         // per-CTA (row, column) slots
  static constexpr int kRing = 8;                // past states a_{n-1..n-8}
  static constexpr int kRedVals = 4;
  static constexpr int kRed = 2 * kRedVals * CS * kWarps;
  static constexpr int kSmemDoubles = 4 * kV + kRing * kSlots + kRed + 4;   // + VC[1], mbarriers
  static_assert(TX % 32 == 0, "column threads must fill warps");
  static_assert((CS * kWarps) % 32 == 0 || CS * kWarps < 32, "reduction layout");
};

__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

// 32-bit shared::cluster addressing (DSMEM stores without generic pointers)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

// mbarrier primitives: the PCG loop's halo exchange and dot-product all-reduce
// deliver their data with st.async into the receiving CTA and signal it on a
// transaction-counting mbarrier there, instead of cluster-wide barriers
// (the band path's protocol, band_path.cu).
__device__ __forceinline__ void cl_mb_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(mb)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void cl_mb_expect(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_mb_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT%=;\n"
      "}\n" ::"r"(smem_addr(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cl_st_async(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(
                   addr),
               "d"(v), "r"(mbar)
               : "memory");
}

template <class C>
struct Thr {
  int x;      // grid column
  int k;      // strip of the band
  int rank;   // CTA rank = band index
  int gy0;    // global grid row of slot 0
  __device__ bool ok(int r, const ClArgs& a) const { return x < a.wd && gy0 + r < a.gh; }
  __device__ int row(int r, const ClArgs& a) const { return (gy0 + r) * a.wd + x; }
  __device__ int vidx(int r) const { return (k * C::R + r + 1) * C::LD + x + 1; }
  __device__ int slot(int r) const { return (k * C::R + r) * C::TX + x; }
};

template <class C>
struct ClOp {
  static constexpr int R = C::R;
  double a[R][7];
  double dinv[R];
  double lf[R - 1];

  __device__ void load(const Thr<C>& th, const ClArgs& A, const double* __restrict__ Ms,
                       const double* __restrict__ Ks, double dt) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool v = th.ok(r, A);
      const int rw = v ? th.row(r, A) : 0;
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        if (j == 1 && r > 0) continue;   // S of slot r = N of slot r-1 (A symmetric)
        const int q = v ? __ldg(A.gpos + (int64_t)j * A.N + rw) : -1;
        a[r][j] = q >= 0 ? op_entry(__ldg(Ms + q), __ldg(Ks + q), dt) : 0.0;
      }
    }
    // block-Jacobi on the thread's R-row strip: B = L D L^T (as GridOp)
    double d = a[0][3];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r > 0) {
        const double nprev = a[r - 1][5];
        lf[r - 1] = (d != 0.0) ? nprev / d : 0.0;
        d = a[r][3] - lf[r - 1] * nprev;
      }
      dinv[r] = (th.ok(r, A) && d != 0.0) ? 1.0 / d : 0.0;
    }
  }
  __device__ void precond(const double (&r_)[R], double (&z)[R]) const {
    double y[R];
    y[0] = r_[0];
#pragma unroll
    for (int r = 1; r < R; ++r) y[r] = fma(-lf[r - 1], y[r - 1], r_[r]);
    z[R - 1] = dinv[R - 1] * y[R - 1];
#pragma unroll
    for (int r = R - 2; r >= 0; --r) z[r] = fma(-lf[r], z[r + 1], dinv[r] * y[r]);
  }
  // the 7 neighbour values (SW,S,W,C,E,N,NE) of each slot
  __device__ static void neighbours(const Thr<C>& th, const double (&v)[R], const double* V,
                                    double (&nb)[R][7]) {
    constexpr int LD = C::LD;
    const int b = th.vidx(0);
    double wr[R], er[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      wr[r] = V[b + r * LD - 1];
      er[r] = V[b + r * LD + 1];
    }
    const double s0 = V[b - LD], sw0 = V[b - LD - 1];
    const double nt = V[b + R * LD], net = V[b + R * LD + 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      nb[r][0] = r > 0 ? wr[r - 1] : sw0;
      nb[r][1] = r > 0 ? v[r - 1] : s0;
      nb[r][2] = wr[r];
      nb[r][3] = v[r];
      nb[r][4] = er[r];
      nb[r][5] = r < R - 1 ? v[r + 1] : nt;
      nb[r][6] = r < R - 1 ? er[r + 1] : net;
    }
  }
  __device__ void apply(const Thr<C>& th, const double (&v)[R], const double* V,
                        double (&out)[R]) const {
    double nb[R][7];
    neighbours(th, v, V, nb);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc0 = a[r][3] * nb[r][3];
      double acc1 = a[r][0] * nb[r][0];
      acc0 = fma(r > 0 ? a[r - 1][5] : a[0][1], nb[r][1], acc0);
      acc1 = fma(a[r][2], nb[r][2], acc1);
      acc0 = fma(a[r][4], nb[r][4], acc0);
      acc1 = fma(a[r][5], nb[r][5], acc1);
      acc0 = fma(a[r][6], nb[r][6], acc0);
      out[r] = acc0 + acc1;
    }
  }
  // out = M v from the stencil-slot layout (M7s = the sample's [7][N] slice):
  // apply_vals' sums with direct, coalesced loads instead of the gpos gather
  // (zero slots add exact zeros)
  __device__ static void apply_m7(const Thr<C>& th, const ClArgs& A, const double* __restrict__ M7s,
                                  const double (&v)[R], const double* V, double (&out)[R]) {
    double nb[R][7];
    neighbours(th, v, V, nb);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if (th.ok(r, A)) {
        const int rw = th.row(r, A);
#pragma unroll
        for (int j = 0; j < 7; ++j) acc = fma(__ldg(M7s + (int64_t)j * A.N + rw), nb[r][j], acc);
      }
      out[r] = acc;
    }
  }
  // out = B v for per-sample CSR values B (the energy, and M a_n once per step)
  __device__ static void apply_vals(const Thr<C>& th, const ClArgs& A,
                                    const double* __restrict__ vals, const double (&v)[R],
                                    const double* V, double (&out)[R]) {
    double nb[R][7];
    neighbours(th, v, V, nb);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if (th.ok(r, A)) {
        const int rw = th.row(r, A);
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          const int q = __ldg(A.gpos + (int64_t)j * A.N + rw);
          if (q >= 0) acc = fma(__ldg(vals + q), nb[r][j], acc);
        }
      }
      out[r] = acc;
    }
  }
};

// Store the thread's R values into the CTA's exchange buffer; the band's first
// / last grid row also into the halo row of the CTA below / above (DSMEM).
template <class C>
__device__ __forceinline__ void publish(const Thr<C>& th, const double (&v)[C::R], double* V,
                                        cg::cluster_group&) {
  const int b = th.vidx(0);
#pragma unroll
  for (int r = 0; r < C::R; ++r) V[b + r * C::LD] = v[r];
  if (th.k == 0 && th.rank > 0)
    st_cluster(map_rank(smem_addr(V + (C::HB + 1) * C::LD + th.x + 1), th.rank - 1), v[0]);
  if (th.k == C::NS - 1 && th.rank < C::CS - 1)
    st_cluster(map_rank(smem_addr(V + th.x + 1), th.rank + 1), v[C::R - 1]);
}

// Cluster all-reduce of NV <= 4 doubles; every thread of every CTA returns
// bitwise identical totals (same partials, same fixed order).
template <class C, int NV>
__device__ __forceinline__ void cl_allsum(double (&v)[NV], double* red, int& par, int rank,
                                          cg::cluster_group& cl) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  constexpr int E = C::CS * C::kWarps;          // partials per value
  double* buf = red + par * (C::kRedVals * E);
  if (lane < C::CS) {
    const uint32_t dst = map_rank(smem_addr(buf + rank * C::kWarps + warp), lane);
#pragma unroll
    for (int k = 0; k < NV; ++k) st_cluster(dst + 8u * (uint32_t)(k * E), v[k]);
  }
  cl_sync();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < (E + 31) / 32; ++e)
      if (e * 32 + lane < E) s += buf[k * E + e * 32 + lane];
    v[k] = s;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  par ^= 1;
}

template <class C>
struct ClShared {
  double* VA;    // exchange: a_n (rhs), x (energy)
  double* VB;    // exchange: initial guess
  double* VC;    // exchange: u (PCG iterations), two buffers alternating by exchange
  uint64_t* mb;  // mbarriers: [0..1] halo rows of VC[b], [2..3] CTA partials of red[b]
  uint32_t ph;   // wait parity bits of the mbarriers
  int hb;        // VC buffer of the current exchange
  int dbg;       // MLMCP_CLUSTER_SYNC=1: cluster barriers around every exchange / all-reduce
  const double* Ms;   // per-sample CSR mass values (M a_n once per step, from L2)
  const double* M7s;  // the same in stencil-slot layout [7][N], or null
  double* ring;  // [kRing][kSlots] past states
  double* red;   // [2][kRedVals][CS][kWarps]
  int par;
};

// u into the next of the two PCG exchange buffers: own rows by plain stores,
// the band's edge rows into the neighbouring CTAs' halo rows by st.async
// counted on their mbarrier; then wait for this CTA's two halo rows.  Every
// buffer is rewritten only after the CTAs reading it have contributed to an
// all-reduce in between.
template <class C>
__device__ __forceinline__ double* cl_exchange(const Thr<C>& th, const double (&v)[C::R],
                                               ClShared<C>& sh) {
  if (sh.dbg) cl_sync();
  sh.hb ^= 1;
  double* V = sh.VC + sh.hb * C::kV;
  uint64_t* mb = sh.mb + sh.hb;
  const int b = th.vidx(0);
  MLMCP_DCHECK(b - C::LD - 1 >= 0 && b + C::R * C::LD + 1 < C::kV);
#pragma unroll
  for (int r = 0; r < C::R; ++r) V[b + r * C::LD] = v[r];
  if (th.k == 0 && th.rank > 0)
    cl_st_async(map_rank(smem_addr(V + (C::HB + 1) * C::LD + th.x + 1), th.rank - 1), v[0],
                map_rank(smem_addr(mb), th.rank - 1));
  if (th.k == C::NS - 1 && th.rank < C::CS - 1)
    cl_st_async(map_rank(smem_addr(V + th.x + 1), th.rank + 1), v[C::R - 1],
                map_rank(smem_addr(mb), th.rank + 1));
  if (threadIdx.x == 0)
    cl_mb_expect(mb, 8u * C::TX * ((th.rank > 0 ? 1u : 0u) + (th.rank < C::CS - 1 ? 1u : 0u)));
  __syncthreads();
  cl_mb_wait(mb, (sh.ph >> sh.hb) & 1u);
  sh.ph ^= 1u << sh.hb;
  if (sh.dbg) cl_sync();
  return V;
}

// Cluster all-reduce of NV <= 4 doubles without a cluster barrier: warp
// butterfly, the CTA's warp partials summed in warp order, the CTA totals
// stored into every CTA by st.async (counted on its mbarrier), the CTA totals
// summed in rank order.  Bitwise identical totals in every thread of every CTA.
template <class C, int NV>
__device__ __forceinline__ void cl_allsum_mb(double (&v)[NV], ClShared<C>& sh, int rank) {
  constexpr int W = C::kWarps, CS = C::CS;
  static_assert((W & (W - 1)) == 0 && W <= 32 && (CS & (CS - 1)) == 0 && CS <= 32, "widths");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  if (sh.dbg) cl_sync();
  double* wp = sh.red + 2 * 4 * CS;          // [4][W]
  double* cp = sh.red + sh.par * 4 * CS;     // [4][CS]
  uint64_t* mb = sh.mb + 2 + sh.par;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) wp[k * W + warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = wp[k * W + (lane & (W - 1))];
#pragma unroll
      for (int off = W / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, W);
      v[k] = s;
    }
    if (lane < CS) {
      const uint32_t dst = map_rank(smem_addr(cp + rank), lane);
      const uint32_t rmb = map_rank(smem_addr(mb), lane);
#pragma unroll
      for (int k = 0; k < NV; ++k) cl_st_async(dst + 8u * (uint32_t)(k * CS), v[k], rmb);
    }
    if (lane == 0) cl_mb_expect(mb, 8u * CS * NV);
  }
  cl_mb_wait(mb, (sh.ph >> (2 + sh.par)) & 1u);
  sh.ph ^= 1u << (2 + sh.par);
  if (sh.dbg) cl_sync();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = cp[k * CS + (lane & (CS - 1))];
#pragma unroll
    for (int off = CS / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, CS);
    v[k] = s;
  }
  sh.par ^= 1;
}

// 1/2 x^T B x over the cluster (every thread receives it)
template <class C>
__device__ __forceinline__ double cl_energy(const Thr<C>& th, const ClArgs& A,
                                            const double (&x)[C::R], const double* vals,
                                            ClShared<C>& sh, cg::cluster_group& cl) {
  publish<C>(th, x, sh.VA, cl);
  cl_sync();
  double bx[C::R];
  ClOp<C>::apply_vals(th, A, vals, x, sh.VA, bx);
  double v[1] = {0.0};
#pragma unroll
  for (int r = 0; r < C::R; ++r) v[0] = fma(x[r], bx[r], v[0]);
  cl_allsum_mb<C, 1>(v, sh, th.rank);
  return 0.5 * v[0];
}

// One implicit-Euler step (M + dt K) a_{n+1} = M a_n + dt*sf*profile, x holds
// the initial guess on entry and a_{n+1} on exit (ie_step of small_path.cu
// with cluster exchanges and reductions).  Returns MLMCP_ST_*.
template <class C>
__device__ __forceinline__ int cl_ie_step(const ClOp<C>& op, const Thr<C>& th, const ClArgs& A,
                                          double (&x)[C::R], const double (&an)[C::R], double sf,
                                          double dt, ClShared<C>& sh, cg::cluster_group& cl,
                                          int& iters) {
  constexpr int R = C::R;
  publish<C>(th, an, sh.VA, cl);
  publish<C>(th, x, sh.VB, cl);
  cl_sync();
  double res[R], u[R], p[R], s[R], w[R];
  double red3[3] = {0.0, 0.0, 0.0};
  {
    double mx[R], ax[R], bv[R];
    if (sh.M7s != nullptr) ClOp<C>::apply_m7(th, A, sh.M7s, an, sh.VA, mx);
    else ClOp<C>::apply_vals(th, A, sh.Ms, an, sh.VA, mx);
    op.apply(th, x, sh.VB, ax);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      res[r] = 0.0;
      bv[r] = 0.0;
      if (th.ok(r, A)) {
        const int rw = th.row(r, A);
        bv[r] = __dadd_rn(mx[r], __dmul_rn(dt, __dmul_rn(sf, __ldg(A.profile + rw))));
        res[r] = bv[r] - ax[r];
      }
    }
    op.precond(bv, u);
#pragma unroll
    for (int r = 0; r < R; ++r) red3[2] = fma(bv[r], u[r], red3[2]);
  }
  op.precond(res, u);
  const double* VU = cl_exchange<C>(th, u, sh);
  op.apply(th, u, VU, w);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    red3[0] += res[r] * u[r];
    red3[1] += w[r] * u[r];
  }
  cl_allsum_mb<C, 3>(red3, sh, th.rank);
  const double gamma = red3[0];
  double delta = red3[1];
  const double bnorm2 = red3[2];
  if (bnorm2 == 0.0) {
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = 0.0;
    return MLMCP_ST_OK;
  }
  const double tol2 = A.rtol2 * bnorm2;
  if (gamma <= tol2) return MLMCP_ST_OK;
  if (!isfinite(gamma)) return MLMCP_ST_NONFINITE;
  if (!(delta > 0.0)) return MLMCP_ST_BREAKDOWN;
  double alpha = gamma * fast_rcp(delta);
  double inv_g = fast_rcp(gamma);
  double c = inv_g * (delta * inv_g);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    p[r] = u[r];
    s[r] = w[r];
    x[r] = fma(alpha, p[r], x[r]);
    res[r] = fma(-alpha, s[r], res[r]);
  }
  int it = 1;
  for (;;) {
    op.precond(res, u);
    const double* VUk = cl_exchange<C>(th, u, sh);
    op.apply(th, u, VUk, w);
    double red2[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      red2[0] = fma(res[r], u[r], red2[0]);
      red2[1] = fma(w[r], u[r], red2[1]);
    }
    cl_allsum_mb<C, 2>(red2, sh, th.rank);
    const double gnew = red2[0];
    delta = red2[1];
    if (gnew <= tol2) break;
    if (!isfinite(gnew)) { iters += it; return MLMCP_ST_NONFINITE; }
    if (it >= A.max_it) { iters += it; return MLMCP_ST_NOCONV; }
    const double beta = gnew * inv_g;
    const double den = fma(-(gnew * gnew), c, delta);
    if (!(den > 0.0)) { iters += it; return MLMCP_ST_BREAKDOWN; }
    alpha = gnew * fast_rcp(den);
    inv_g = fast_rcp(gnew);
    c = inv_g * (den * inv_g);
    op.precond(res, u);
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

// extrapolation weights: a_{n+1} ~ sum_j c[p][j] a_{n-j}, c[p][j] = (-1)^j C(p+1, j+1)
__constant__ double c_cl_extrap[8][8] = {
    {1, 0, 0, 0, 0, 0, 0, 0},
    {2, -1, 0, 0, 0, 0, 0, 0},
    {3, -3, 1, 0, 0, 0, 0, 0},
    {4, -6, 4, -1, 0, 0, 0, 0},
    {5, -10, 10, -5, 1, 0, 0, 0},
    {6, -15, 20, -15, 6, -1, 0, 0},
    {7, -21, 35, -35, 21, -7, 1, 0},
    {8, -28, 56, -70, 56, -28, 8, -1}};

// x <- order-p extrapolation of a_n (x on entry) and the past states in the ring
template <class C>
__device__ __forceinline__ void cl_guess(const Thr<C>& th, double (&x)[C::R], const double* ring,
                                         int step, int p) {
  constexpr int kR = C::kRing;
  if (p <= 0) return;
#pragma unroll
  for (int r = 0; r < C::R; ++r) {
    double g = c_cl_extrap[p][0] * x[r];
    for (int j = 1; j <= p; ++j)
      g = fma(c_cl_extrap[p][j], ring[((step - j) & (kR - 1)) * C::kSlots + th.slot(r)], g);
    x[r] = g;
  }
}

template <class C>
__global__ void __launch_bounds__(C::kThreads, 1) cluster_propagate_kernel(ClArgs a) {
  constexpr int R = C::R;
  extern __shared__ __align__(16) double smem[];
  __shared__ int live;
  cg::cluster_group cl = cg::this_cluster();
  Thr<C> th;
  th.rank = (int)cl.block_rank();
  th.x = threadIdx.x % C::TX;
  th.k = threadIdx.x / C::TX;
  th.gy0 = th.rank * C::HB + th.k * R;
  const mlmcp_task t = a.tasks[blockIdx.x / C::CS];
  const int64_t t_start = global_ns();
  ClShared<C> sh;
  sh.VA = smem;
  sh.VB = sh.VA + C::kV;
  sh.VC = sh.VB + C::kV;
  sh.ring = sh.VC + 2 * C::kV;
  sh.red = sh.ring + C::kRing * C::kSlots;
  sh.mb = reinterpret_cast<uint64_t*>(sh.red + C::kRed);
  sh.ph = 0u;
  sh.hb = 1;
  sh.par = 0;
  sh.dbg = a.dbg_sync;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) cl_mb_init(sh.mb + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < 4 * C::kV; i += C::kThreads) smem[i] = 0.0;
  if (th.rank == 0 && threadIdx.x == 0) {
    const int lv = (a.active == nullptr || t.group < 0)
                       ? 1
                       : (*((volatile const int32_t*)a.active + t.group) != 0);
    for (int c = 0; c < C::CS; ++c) *cl.map_shared_rank(&live, c) = lv;
  }
  cl_sync();   // zeroed buffers and the live flag visible cluster-wide
  if (!live) return;   // cluster-uniform

  const double* Ms = a.M + (int64_t)t.sample * a.nnz;
  const double* Ks = a.K + (int64_t)t.sample * a.nnz;
  ClOp<C> op;
  op.load(th, a, Ms, Ks, t.dt);
  sh.Ms = Ms;
  sh.M7s = a.M7 ? a.M7 + (int64_t)t.sample * 7 * a.N : nullptr;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool v = th.ok(r, a);
    const int rw = v ? th.row(r, a) : 0;
    x[r] = v ? __ldcg(a.xbuf + t.x_in + rw) : 0.0;
    if (t.traj >= 0 && v) a.xbuf[t.traj + rw] = x[r];
  }
  const int max_order = (t.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : a.order;
  int iters = 0, code = MLMCP_ST_OK, fail_step = 0;
  double acc = 0.0;
  for (int step = 0; step < t.n_steps; ++step) {
    const int64_t g = t.k0 + step + 1;
    const double sf = sin(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)));
    double an[R];
#pragma unroll
    for (int r = 0; r < R; ++r) an[r] = x[r];
    cl_guess<C>(th, x, sh.ring, step, min(step, max_order));
    // a_n joins the ring (after the guess read the oldest entry)
#pragma unroll
    for (int r = 0; r < R; ++r) sh.ring[(step & (C::kRing - 1)) * C::kSlots + th.slot(r)] = an[r];
    code = cl_ie_step<C>(op, th, a, x, an, sf, t.dt, sh, cl, iters);
    if (code != MLMCP_ST_OK) { fail_step = step; break; }
    if (t.traj >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (th.ok(r, a)) a.xbuf[t.traj + (int64_t)(step + 1) * a.N + th.row(r, a)] = x[r];
    }
    if (g > t.qoi_from && t.qoi_mode == MLMCP_QOI_SUM_ENERGY)
      acc += cl_energy<C>(th, a, x, Ks, sh, cl);
  }
  if (t.x_out >= 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (th.ok(r, a)) a.xbuf[t.x_out + th.row(r, a)] = x[r];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY && t.qoi_slot >= 0)
    acc = cl_energy<C>(th, a, x, Ks, sh, cl);
  if (th.rank == 0 && threadIdx.x == 0) {
    if (t.qoi_slot >= 0 && t.qoi_mode != MLMCP_QOI_NONE) a.qoi[t.qoi_slot] = acc;
    if (a.iters != nullptr && t.slot >= 0) atomicAdd(a.iters + t.slot, iters);
    add_elapsed(a.elapsed, t.slot, t_start);
    if (code != MLMCP_ST_OK) {
      write_status(a.status, t.slot, code, fail_step, t.tag, t.tag);
      if (a.active != nullptr && t.group >= 0) const_cast<int32_t*>(a.active)[t.group] = 0;
    }
  }
  cl_sync();   // no CTA leaves while another may still address its shared memory
}


// Parareal coarse sweep on the cluster path (parareal.py:168-178): one
// cluster per Parareal sample walks the slices n = k .. m-1 of iteration k:
// propagate U_{n-1} over slice n with the coarse step (the operator at dt_c
// stays in registers for the whole sweep), then
//   k == 1: U_n = C_{n-1} = c;   k >= 2: U_n = (F_n + c) - C_{n-1}, C_{n-1} = c
// (the arithmetic of correct_kernel).  A failed coarse solve records
// (code, step, interval n, iteration k) and deactivates the sample, as the
// streaming sweep's coarse_status_kernel.  Replaces ~30 launches per slice of
// the streaming sweep with one launch per sweep.
struct ClCoarse {
  int k, m;
  double dt_c, t0;
  const int64_t* slice_k0;
  const int32_t* slice_steps;
  double* U;          // [S][m+1][N]
  const double* F;    // [S][m+1][N]
  double* C;          // [S][m][N]
};

template <class C>
__global__ void __launch_bounds__(C::kThreads, 1) cluster_coarse_kernel(ClArgs a, ClCoarse cc) {
  constexpr int R = C::R;
  extern __shared__ __align__(16) double smem[];
  __shared__ int live;
  cg::cluster_group cl = cg::this_cluster();
  Thr<C> th;
  th.rank = (int)cl.block_rank();
  th.x = threadIdx.x % C::TX;
  th.k = threadIdx.x / C::TX;
  th.gy0 = th.rank * C::HB + th.k * R;
  const int s = blockIdx.x / C::CS;
  ClShared<C> sh;
  sh.VA = smem;
  sh.VB = sh.VA + C::kV;
  sh.VC = sh.VB + C::kV;
  sh.ring = sh.VC + 2 * C::kV;
  sh.red = sh.ring + C::kRing * C::kSlots;
  sh.mb = reinterpret_cast<uint64_t*>(sh.red + C::kRed);
  sh.ph = 0u;
  sh.hb = 1;
  sh.par = 0;
  sh.dbg = a.dbg_sync;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) cl_mb_init(sh.mb + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < 4 * C::kV; i += C::kThreads) smem[i] = 0.0;
  if (th.rank == 0 && threadIdx.x == 0) {
    const int lv = *((volatile const int32_t*)a.active + s) != 0;
    for (int c = 0; c < C::CS; ++c) *cl.map_shared_rank(&live, c) = lv;
  }
  cl_sync();
  if (!live) return;
  const int64_t N = a.N;
  const double* Ms = a.M + (int64_t)s * a.nnz;
  const double* Ks = a.K + (int64_t)s * a.nnz;
  ClOp<C> op;
  op.load(th, a, Ms, Ks, cc.dt_c);
  sh.Ms = Ms;
  sh.M7s = nullptr;
  double* Us = cc.U + (int64_t)s * (cc.m + 1) * N;
  const double* Fs = cc.F + (int64_t)s * (cc.m + 1) * N;
  double* Cs = cc.C + (int64_t)s * cc.m * N;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    x[r] = th.ok(r, a) ? __ldcg(Us + (int64_t)(cc.k - 1) * N + th.row(r, a)) : 0.0;
  int iters = 0;
  for (int n = cc.k; n < cc.m; ++n) {
    const int n_steps = cc.slice_steps[n - 1];
    const int64_t k0 = cc.slice_k0[n - 1];
    int code = MLMCP_ST_OK, fail_step = 0;
    for (int step = 0; step < n_steps; ++step) {
      const int64_t g = k0 + step + 1;
      const double sf = sin(__dmul_rn(a.omega, grid_time(cc.t0, g, cc.dt_c)));
      double an[R];
#pragma unroll
      for (int r = 0; r < R; ++r) an[r] = x[r];
      cl_guess<C>(th, x, sh.ring, step, min(step, a.order));
#pragma unroll
      for (int r = 0; r < R; ++r) sh.ring[(step & (C::kRing - 1)) * C::kSlots + th.slot(r)] = an[r];
      code = cl_ie_step<C>(op, th, a, x, an, sf, cc.dt_c, sh, cl, iters);
      if (code != MLMCP_ST_OK) { fail_step = step; break; }
    }
    if (code != MLMCP_ST_OK) {   // cluster-uniform (scalars are identical in every CTA)
      if (th.rank == 0 && threadIdx.x == 0) {
        if (a.status[(int64_t)s * kStatusInts] == MLMCP_ST_OK)
          write_status(a.status, s, code, fail_step, n, cc.k);
        const_cast<int32_t*>(a.active)[s] = 0;
      }
      break;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!th.ok(r, a)) continue;
      const int64_t i = th.row(r, a);
      const double c = x[r];
      const double u = cc.k == 1 ? c : (Fs[(int64_t)n * N + i] + c) - Cs[(int64_t)(n - 1) * N + i];
      Us[(int64_t)n * N + i] = u;
      Cs[(int64_t)(n - 1) * N + i] = c;
      x[r] = u;
    }
  }
  cl_sync();   // no CTA leaves while another may still address its shared memory
}

// per-sample mass values into the stencil-slot layout [S][7][N] (SW..NE; 0 where
// the neighbour is a Dirichlet node)
__global__ void m7_kernel(int S, int N, int64_t nnz, const int32_t* gpos, const double* M,
                          double* M7) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)7 * N) return;
  const int s = blockIdx.y;
  const int q = gpos[i];
  M7[(int64_t)s * 7 * N + i] = q >= 0 ? M[(int64_t)s * nnz + q] : 0.0;
}

// 128 column threads x 4 strips of 4 rows, 8 CTAs: grids up to 128 x 128
using Cfg128 = Cfg<4, 128, 4, 8>;

template <class C>
int launch(const ClArgs& a, int n_tasks, cudaStream_t stream) {
  const size_t smem = sizeof(double) * C::kSmemDoubles;
  static bool attr_done = false;
  if (!attr_done) {
    MLMCP_CUDA_CHECK(cudaFuncSetAttribute(cluster_propagate_kernel<C>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_tasks * C::CS));
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, cluster_propagate_kernel<C>, a));
  MLMCP_LAUNCH_CHECK("cluster_propagate_kernel");
  return MLMCP_OK;
}

int cluster_dbg_sync() {
  const char* e = getenv("MLMCP_CLUSTER_SYNC");
  return (e && atoi(e) != 0) ? 1 : 0;
}

int order_pref() {
  const char* e = getenv("MLMCP_CLUSTER_ORDER");
  const int o = e ? atoi(e) : 7;   // higher orders pay: smooth states in time
  return std::max(0, std::min(o, 7));
}

}  // namespace

bool cluster_usable(const Ctx* ctx) {
  // MLMCP_STREAM_IMPL: 1 two-launch, 2 cooperative, 3 cluster, 4 tile, 5 band, default
  // auto (cluster when it fits)
  const char* e = getenv("MLMCP_STREAM_IMPL");
  const int impl = e ? atoi(e) : 0;
  if (impl == 1 || impl == 2 || impl == 4 || impl == 5) return false;
  return ctx->cl_wd > 0 && ctx->cl_wd <= Cfg128::TX &&
         ctx->cl_h <= Cfg128::CS * Cfg128::HB;
}

int cluster_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, int S, const double* M,
                      const double* K, const double* profile, double omega, double rtol,
                      int max_it, double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                      const int32_t* active, int64_t* elapsed, void* ws, size_t ws_bytes,
                      cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  ClArgs a;
  a.M7 = nullptr;
  a.dbg_sync = cluster_dbg_sync();
  if (ws != nullptr && ws_bytes >= sizeof(double) * (size_t)S * 7 * (size_t)ctx->n) {
    double* m7 = static_cast<double*>(ws);
    m7_kernel<<<dim3((unsigned)((7 * (int64_t)ctx->n + 255) / 256), (unsigned)S), 256, 0, stream>>>(
        S, ctx->n, ctx->nnz, ctx->cl_pos, M, m7);
    MLMCP_LAUNCH_CHECK("m7_kernel");
    a.M7 = m7;
  }
  a.tasks = tasks;
  a.N = ctx->n;
  a.wd = ctx->cl_wd;
  a.gh = ctx->cl_h;
  a.nnz = ctx->nnz;
  a.gpos = ctx->cl_pos;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.order = order_pref();
  a.xbuf = xbuf;
  a.qoi = qoi;
  a.iters = iters;
  a.status = status;
  a.active = active;
  a.elapsed = elapsed;
  return launch<Cfg128>(a, n_tasks, stream);
}


int cluster_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                            const double* profile, double omega, double dt_c, double t0,
                            const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                            int max_it, double* U, const double* F, double* C, int32_t* status,
                            const int32_t* active, cudaStream_t stream) {
  if (S == 0 || k >= m) return MLMCP_OK;
  using Cf = Cfg128;
  ClArgs a{};
  a.M7 = nullptr;
  a.dbg_sync = cluster_dbg_sync();
  a.N = ctx->n;
  a.wd = ctx->cl_wd;
  a.gh = ctx->cl_h;
  a.nnz = ctx->nnz;
  a.gpos = ctx->cl_pos;
  a.M = M;
  a.K = K;
  a.profile = profile;
  a.omega = omega;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.order = order_pref();
  a.status = status;
  a.active = active;
  ClCoarse cc{k, m, dt_c, t0, slice_k0, slice_steps, U, F, C};
  const size_t smem = sizeof(double) * Cf::kSmemDoubles;
  static bool attr_done = false;
  if (!attr_done) {
    MLMCP_CUDA_CHECK(cudaFuncSetAttribute(cluster_coarse_kernel<Cf>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(S * Cf::CS));
  cfg.blockDim = dim3(Cf::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cf::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, cluster_coarse_kernel<Cf>, a, cc));
  MLMCP_LAUNCH_CHECK("cluster_coarse_kernel");
  return MLMCP_OK;
}

}  // namespace mlmcp
