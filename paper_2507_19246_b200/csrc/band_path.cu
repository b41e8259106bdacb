// band_path.cu — cluster-resident implicit Euler for region-linear structured
// grids of up to 256 x 256 interior points (config 2's 256^2 mesh: 65,025
// unknowns per sample), one 16-CTA thread-block cluster per task.
//
// Same method and step semantics as the HBM-streaming tile path
// (stream_path.cu; reference timeint.py:88-128): per step the periodic
// steady-state predictor plus the least-squares transient guess (ring of 8 past
// transients), the rhs b = M a_n + dt sin(wt) profile, and a Chronopoulos-Gear
// PCG solve with the stopping rule r.B^-1.r <= rtol^2 b.B^-1.b.  What changes
// is where the PCG vectors live: a cluster of 16 CTAs (one per SM, 256 threads
// each) owns one task for all its steps; CTA c holds the band of grid rows
// [16c, 16c+16) and each thread a column strip of 16 rows, so the PCG vectors
// p, s, r, w stay in registers and x in shared memory for the whole solve — a
// PCG iteration moves no global memory at all (the tile path streams 64 B per
// point and iteration).  Global traffic per step is the guess: 7 ring reads and
// 1 ring write per point, on a ring that stays L2-resident (7 concurrent
// clusters x 4.2 MB).
//   * operator: the task's stencil of each point class (Ctx::rckey) formed once
//     per task into shared memory (A, M and K rows, region_stencil of
//     stream_path.cu's arithmetic); a thread keeps the row of its strip's class
//     in registers and reloads it only where the class changes (Row7);
//   * preconditioner: 16-row strip block-Jacobi (L D L^T of each strip), one
//     set of factors per strip signature (class sequence) in shared memory;
//   * the task's periodic steady state in shared memory for all its steps;
//   * neighbour values through a shared-memory exchange frame; a band's first
//     and last grid rows also go straight into the neighbouring CTAs' frames
//     (st.async, counted on a transaction mbarrier there); the rows that need
//     no other band's values are formed before the wait for the halo rows;
//   * dot products: warp butterfly, fixed-order sum of the CTA's 8 warp
//     partials, the 16 CTA partials stored into every CTA (st.async on an
//     mbarrier), fixed-order sum — bitwise identical scalars in every CTA,
//     hence one control flow for the whole cluster; no cluster barrier in the
//     step loop.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <vector>

#include "mlmcp_internal.cuh"

namespace mlmcp {
namespace {

namespace cg = cooperative_groups;

constexpr int kR = 16;                   // grid rows per thread strip (the CTA's band)
constexpr int kTX = 256;                 // column threads (grid columns per cluster)
constexpr int kNS = 1;                   // strips per CTA
constexpr int kCS = 16;                  // CTAs per cluster
constexpr int kNT = kTX * kNS;           // 256 threads
constexpr int kWarps = kNT / 32;
constexpr int kHB = kR * kNS;            // 16 grid rows per CTA
constexpr int kLD = kTX + 2;             // exchange-buffer row stride
constexpr int kV = (kHB + 2) * kLD;      // one exchange buffer
constexpr int kSlots = kHB * kTX;        // (row, column) slots per CTA
constexpr int kRing = 8;                 // past transients (extrapolation order <= 7)
#ifndef MLMCP_BAND_GB
#define MLMCP_BAND_GB 8
#endif
constexpr int kGB = MLMCP_BAND_GB;       // guess rows whose ring loads are in flight together
constexpr int kBandPts = kCS * kHB * kTX;  // ring slot pitch: rows of kTX points (compile-time offsets)
constexpr int kMaxC = 256;               // point classes
constexpr int kMaxSig = 32;              // distinct strip signatures (class sequences) per CTA
constexpr int kPF = (2 * kR - 1) * kMaxSig;   // strip factors, one set per signature
constexpr int kTabW = 24;                // per class: A (7 + pad), M (7 + pad), K (7 + pad)
// shared memory (doubles): VA, VC[2], x, strip factors, class table, reduction
// buffers, mbarriers
constexpr int kRedD = 2 * 4 * kCS + 4 * kWarps;

__constant__ double c_bd_extrap[8][8] = {
    {1, 0, 0, 0, 0, 0, 0, 0},
    {2, -1, 0, 0, 0, 0, 0, 0},
    {3, -3, 1, 0, 0, 0, 0, 0},
    {4, -6, 4, -1, 0, 0, 0, 0},
    {5, -10, 10, -5, 1, 0, 0, 0},
    {6, -15, 20, -15, 6, -1, 0, 0},
    {7, -21, 35, -35, 21, -7, 1, 0},
    {8, -28, 56, -70, 56, -28, 8, -1}};
// least-squares degree-6 fit through the last 8 transients (stream_path.cu)
__constant__ double c_bd_ls68[8] = {49.0 / 8, -119.0 / 8, 133.0 / 8, -35.0 / 8,
                                    -77.0 / 8, 91.0 / 8, -41.0 / 8, 7.0 / 8};
// degree-5 / degree-4 fits through the same 8 transients.  The degree trades
// truncation error against the amplification of the previous solves' errors
// (sum |w| = 69 / 25.5 / 11.2 for degrees 6 / 5 / 4): measured PCG iterations
// per step at dt = T/64: 3.04 / 4.30 / 6.32, T/128: 3.21 / 3.57 / 5.76, T/256:
// 2.82 / 2.56 / 3.44, T/512: 2.71 / 2.17 / 2.29 — degree 6 up to 192 steps per
// period, degree 5 beyond (MLMCP_BAND_LSDEG = 4 / 5 / 6 forces one, A/B)
__constant__ double c_bd_ls58[8] = {36.0 / 8, -54.0 / 8, 16.0 / 8, 30.0 / 8,
                                    -12.0 / 8, -26.0 / 8, 24.0 / 8, -6.0 / 8};
__constant__ double c_bd_ls48[8] = {175.0 / 56, -125.0 / 56, -75.0 / 56, 45.0 / 56,
                                    81.0 / 56, 5.0 / 56, -85.0 / 56, 35.0 / 56};

// MLMCP_BAND_PROF=1: clock64 cycles of the step phases in CTA 0 of the first
// cluster (trig + sync, guess, step start incl. its all-reduce, PCG loop)
__device__ unsigned long long g_band_prof[16];   // [8..13]: PCG-iteration phases (prof bit 1)
#define BD_PROF(i, t0)                                                              \
  do {                                                                            \
    if (kProf && (a.prof & 1) && blockIdx.x == 0 && threadIdx.x == 0) {                 \
      const long long t1_ = clock64();                                            \
      g_band_prof[i] += (unsigned long long)(t1_ - (t0));                         \
      (t0) = t1_;                                                                 \
    }                                                                             \
  } while (0)

// PCG-iteration phases: compiled in only with -DMLMCP_BAND_PROF2 (the probes
// split the iteration into basic blocks)
#ifdef MLMCP_BAND_PROF2
#define BD_PROF2(i, t0)                                                             \
  do {                                                                            \
    if ((a.prof & 2) && blockIdx.x == 0 && threadIdx.x == 0) {                          \
      const long long t1_ = clock64();                                            \
      g_band_prof[i] += (unsigned long long)(t1_ - (t0));                         \
      (t0) = t1_;                                                                 \
    }                                                                             \
  } while (0)
#define BD_PROF2_T0(t) long long t = clock64()
#else
#define BD_PROF2(i, t0) do { } while (0)
#define BD_PROF2_T0(t) do { } while (0)
#endif

struct BdArgs {
  const mlmcp_task* tasks;
  int N, wd, gh;
  const uint8_t* rcls;
  const uint32_t* rckey;
  int rC;
  const double* rpar;      // [S][R][2] (sigma_r masked, nu_r)
  int R;
  double rmw[12], rkw[12];
  const double* profile;
  const double* xss;       // [slots][2][N] periodic steady states, or null
  double omega, rtol2;
  int max_it;
  int order;
  int ls_on;
  double* ring;            // [T][kRing][kBandPts], point (gx, gy) at gy * kTX + gx
  double* xbuf;
  double* qoi;
  int32_t* iters;
  int32_t* status;
  const int32_t* active;
  int64_t* elapsed;
  int prof;
  int dbg_sync;            // MLMCP_BAND_SYNC=1: cluster barriers around every exchange / all-reduce
};

__device__ __forceinline__ void bd_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bd_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bd_sync() {
  bd_arrive();
  bd_wait();
}
__device__ __forceinline__ uint32_t bd_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t bd_mapa(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// mbarrier primitives: the PCG loop's halo exchange and dot-product all-reduce
// signal completion through transaction-counting mbarriers in the receiving
// CTA (st.async ... complete_tx) instead of cluster-wide barriers.
__device__ __forceinline__ void mb_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bd_smem(mb)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bd_smem(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT%=;\n"
      "}\n" ::"r"(bd_smem(mb)),
      "r"(parity)
      : "memory");
}
// 8-byte store into another CTA's shared memory, counted on its mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(
                   addr),
               "d"(v), "r"(mbar)
               : "memory");
}

// device code: production (bd0) and barrier-serialised debug (bd1) instantiations
namespace bd0 {
constexpr bool kDbg = false, kProf = false;
#include "band_kernel.cuh"
}  // namespace bd0
namespace bd1 {
constexpr bool kDbg = true, kProf = false;
#include "band_kernel.cuh"
}  // namespace bd1
namespace bd2 {   // MLMCP_BAND_PROF=1: per-phase cycle probes
constexpr bool kDbg = false, kProf = true;
#include "band_kernel.cuh"
}  // namespace bd2

size_t band_smem_bytes(int n_classes) {
  return sizeof(double) * (3 * kV + kSlots + kPF + 2 * kSlots + kTabW * n_classes + kRedD + 5);
}

}  // namespace

// MLMCP_BAND=0 keeps 256^2 region grids on the tile path (A/B)
bool band_usable(const Ctx* ctx) {
  const char* e = getenv("MLMCP_BAND");
  if (e && atoi(e) == 0) return false;
  const char* s = getenv("MLMCP_STREAM_IMPL");   // 5: the band path also on <= 128^2 grids
  if (s && atoi(s) != 0 && atoi(s) != 5) return false;
  return ctx->rcls != nullptr && ctx->rC <= kMaxC && ctx->cl_wd > 0 && ctx->cl_wd <= kTX &&
         ctx->cl_h <= kCS * kHB && band_smem_bytes(ctx->rC) <= 227 * 1024 &&
         ctx->band_sigs > 0 && ctx->band_sigs <= kMaxSig;
}

// The largest number of distinct strip signatures (16 row classes + validity
// of a column's strip) in any 16-row band of the grid; 0 when the grid does
// not fit the band decomposition.  Host side, once per region grid.
int band_max_signatures(const uint8_t* cls, int wd, int gh) {
  if (cls == nullptr || wd <= 0 || wd > kTX || gh <= 0 || gh > kCS * kHB) return 0;
  int worst = 0;
  for (int band = 0; band * kHB < gh; ++band) {
    std::vector<std::array<int, kR>> sigs;
    for (int x = 0; x < kTX; ++x) {
      std::array<int, kR> sg;
      for (int r = 0; r < kR; ++r) {
        const int gy = band * kHB + r;
        sg[r] = (x < wd && gy < gh) ? (int)cls[(size_t)gy * wd + x] : -1;
      }
      if (std::find(sigs.begin(), sigs.end(), sg) == sigs.end()) sigs.push_back(sg);
    }
    worst = std::max(worst, (int)sigs.size());
  }
  return worst;
}

size_t band_ring_bytes(int n_tasks) {
  return sizeof(double) * (size_t)n_tasks * kRing * kBandPts;
}

int band_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* rpar,
                   const double* profile, double omega, double rtol, int max_it, int order,
                   int ls_on, const double* xss, double* ring, double* xbuf, double* qoi,
                   int32_t* iters, int32_t* status, const int32_t* active, int64_t* elapsed,
                   cudaStream_t stream) {
  if (n_tasks == 0) return MLMCP_OK;
  BdArgs a;
  a.tasks = tasks;
  a.N = ctx->n;
  a.wd = ctx->cl_wd;
  a.gh = ctx->cl_h;
  a.rcls = ctx->rcls;
  a.rckey = ctx->rckey;
  a.rC = ctx->rC;
  a.rpar = rpar;
  a.R = ctx->rR;
  for (int i = 0; i < 12; ++i) {
    a.rmw[i] = ctx->rmw[i];
    a.rkw[i] = ctx->rkw[i];
  }
  a.profile = profile;
  a.xss = xss;
  a.omega = omega;
  a.rtol2 = rtol * rtol;
  a.max_it = max_it;
  a.order = std::max(0, std::min(order, kRing - 1));
  a.ls_on = ls_on;
  if (const char* ld = getenv("MLMCP_BAND_LSDEG")) {
    const int d = atoi(ld);
    if (ls_on && d >= 4 && d <= 6) a.ls_on = d;
  }
  a.ring = ring;
  a.xbuf = xbuf;
  a.qoi = qoi;
  a.iters = iters;
  a.status = status;
  a.active = active;
  a.elapsed = elapsed;
  const char* pe = getenv("MLMCP_BAND_PROF");
  a.prof = pe ? atoi(pe) : 0;   // bit 0: phase cycles
  const char* ds = getenv("MLMCP_BAND_SYNC");
  a.dbg_sync = (ds && atoi(ds) != 0) ? 1 : 0;
  const size_t smem = band_smem_bytes(a.rC);
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    for (auto k : {bd0::band_propagate_kernel, bd1::band_propagate_kernel,
                   bd2::band_propagate_kernel}) {
      MLMCP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem));
      MLMCP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    attr_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_tasks * kCS));
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // mlmcp_stream_timing: device time of the launch (CUDA events on its stream)
  if (ctx->time_iters) MLMCP_CUDA_CHECK(cudaEventRecord(ctx->iter_ev[0], stream));
  // MLMCP_BAND_SYNC=1: the instantiation with a cluster barrier before and
  // after every exchange and all-reduce (bd1), otherwise the production kernel
  MLMCP_CUDA_CHECK(cudaLaunchKernelEx(&cfg,
                                      a.dbg_sync ? bd1::band_propagate_kernel
                                      : a.prof   ? bd2::band_propagate_kernel
                                                 : bd0::band_propagate_kernel,
                                      a));
  MLMCP_LAUNCH_CHECK("band_propagate_kernel");
  if (ctx->time_iters) {
    MLMCP_CUDA_CHECK(cudaEventRecord(ctx->iter_ev[1], stream));
    MLMCP_CUDA_CHECK(cudaEventSynchronize(ctx->iter_ev[1]));
    float ms = 0.0f;
    MLMCP_CUDA_CHECK(cudaEventElapsedTime(&ms, ctx->iter_ev[0], ctx->iter_ev[1]));
    ctx->iter_ms += ms;
    ctx->iter_launches += 1;
  }
  if (a.prof & 3) {
    unsigned long long h[16];
    MLMCP_CUDA_CHECK(cudaMemcpyFromSymbol(h, g_band_prof, sizeof(h)));
    fprintf(stderr, "band prof cycles: trig %llu guess %llu stepstart+ie %llu pcg %llu tail %llu\n",
            h[0], h[1], h[2], h[3], h[4]);
    if (a.prof & 2)
      fprintf(stderr, "band prof pcg phases: precond %llu exchange %llu apply+dots %llu "
              "allsum %llu update %llu\n", h[8], h[9], h[10], h[11], h[12]);
  }
  return MLMCP_OK;
}

}  // namespace mlmcp
