// mlmcp_internal.cuh — shared internals of libmlmcp.so (sm_100a).
//
// Numerical contract shared by every kernel (matches the reference's
// arithmetic where it is observable, timeint.py:65,78-85,108-110):
//   operator  A_q = M_q + dt*K_q      (rounded product, then rounded sum)
//   grid      t_g = t_base + (double)g * dt
//   forcing   dt * (sin(omega*t_g) * profile_i),  omega = (2*pi)*f on host
//   rhs       b_i = (M x)_i + forcing_i
// All reductions are deterministic (fixed warp-butterfly + fixed cross-warp
// order), so every per-task result is bitwise independent of batch
// composition, launch order and GPU count.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/mlmcp.h"

namespace mlmcp {

constexpr int kMaxNz = 8;         // widest CSR row the kernels accept
constexpr int kStatusInts = 4;    // status[4*slot + {code, step, interval, iteration}]
constexpr int kSmallMaxRows = 1024;  // one row per thread, <=1024 threads

struct Ctx {
  int device = 0;
  int n = 0;            // rows
  int nnz = 0;
  int max_row_nnz = 0;
  int path = 0;         // 0 auto, 1 small, 2 streaming, 3 direct
  int32_t* row_ptr = nullptr;   // device [n+1]
  int32_t* col = nullptr;       // device [nnz]
  int32_t* ell_col = nullptr;   // device [max_row_nnz][n], padded with the row itself
  int32_t* ell_pos = nullptr;   // device [max_row_nnz][n], CSR position or -1
  // uniform-offset stencil view of the pattern (every col - row lies in a set
  // of <= 8 offsets): structured FE meshes, banded models.  stencil_w == 0
  // when the pattern is not a stencil.
  int stencil_w = 0;
  int stencil_off[kMaxNz] = {0};
  int stencil_pad = 0;          // max |offset|
  int32_t* stencil_pos = nullptr;  // device [stencil_w][n]: CSR position or -1
  // 2D grid view (structured 7-point FE stencil on a wd x gh interior grid,
  // row = y*wd + x, neighbours (dx,dy) in {(0,0),(+-1,0),(0,+-1),(1,1),(-1,-1)}),
  // wd <= 32 and gh <= 32: the grid-tiled SM-resident kernel applies.
  int grid_wd = 0;
  int grid_h = 0;
  int32_t* grid_pos = nullptr;     // device [7][n] in order SW,S,W,C,E,N,NE: CSR position or -1
  // the same 2D grid view for larger grids (wd, gh <= 256): the cluster path
  int cl_wd = 0;
  int cl_h = 0;
  int32_t* cl_pos = nullptr;       // device [7][n], as grid_pos
  // assembly gather map
  int n_elem = 0;
  int n_contrib = 0;
  int32_t* cptr = nullptr;
  int32_t* celem = nullptr;
  double* cmw = nullptr;
  double* ckw = nullptr;
  // region-linear operator description (mlmcp_ctx_set_region_grid): the tile
  // kernels compute the operator from per-sample region parameters
  // point classes: every interior point maps to one of rC distinct
  // (six triangle regions, Dirichlet-neighbour mask) keys; the tile kernels
  // form one stencil per class and task in shared memory
  uint8_t* rcls = nullptr;         // device [n] class of each point
  uint32_t* rckey = nullptr;       // device [rC] code (24 bits) | neighbour mask << 24
  int rC = 0;
  int rR = 0;
  int band_sigs = 0;               // most distinct strip signatures in a 16-row band (band path)
  double rmw[12] = {0}, rkw[12] = {0};
  // pinned host counters for the streaming path
  int32_t* host_counters = nullptr;
  // grid-barrier words of the cooperative path (zeroed at creation)
  unsigned int* grid_bar = nullptr;
  // graph-driven step loop of the streaming path: capture streams and the
  // executable graph (updated in place from call to call)
  cudaStream_t cap_stream[3] = {nullptr, nullptr, nullptr};
  cudaGraphExec_t step_exec = nullptr;
  // mlmcp_stream_timing: device time of the PCG-iteration launches
  int time_iters = 0;
  double iter_ms = 0.0;
  int64_t iter_launches = 0;
  cudaEvent_t iter_ev[2] = {nullptr, nullptr};
};

void set_error(const std::string& msg);
void count_launch(uint64_t n = 1);
int cuda_fail(cudaError_t err, const char* what);

#define MLMCP_CUDA_CHECK(call)                                   \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::mlmcp::cuda_fail(_e, #call); \
  } while (0)

#define MLMCP_LAUNCH_CHECK(what)                                 \
  do {                                                           \
    ::mlmcp::count_launch();                                     \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::mlmcp::cuda_fail(_e, what);  \
  } while (0)

// Device-side bounds / invariant checks of the checked build (make checked:
// -DMLMCP_CHECKED, libmlmcp_checked.so).  compute-sanitizer is not available on
// the GPU pool, so the GPU suite runs once against this build (scripts/
// checked_suite.sh): a failed check prints its location and traps the kernel.
#ifdef MLMCP_CHECKED
#include <cstdio>
#define MLMCP_DCHECK(c)                                                                  \
  do {                                                                                   \
    if (!(c)) {                                                                          \
      printf("MLMCP_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x, #c);                                    \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define MLMCP_DCHECK(c) \
  do {                  \
  } while (0)
#endif

// ------------------------------------------------------------------ device
// Reciprocal to ~1 ulp: MUFU approximation + two Newton steps (no slow-path
// branch, so it schedules freely; deterministic).
__device__ __forceinline__ double fast_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Block-wide all-reduce of NV doubles; every thread receives bitwise identical
// totals (xor butterflies are commutative per pair; the cross-warp stage reads
// one shared copy).  `red` holds 2*4*32 doubles, `par` alternates buffers so
// back-to-back calls need no extra barrier.  MAXWARPS (power of two >= the
// block's warp count) bounds the cross-warp butterfly depth.
template <int NV, int MAXWARPS = 32>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* red, int& par) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  double* buf = red + par * (4 * 32);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) buf[k * 32 + warp] = v[k];
  }
  __syncthreads();
  // every group of MAXWARPS lanes reads the same partials, so the shortened
  // butterfly leaves all 32 lanes with bitwise identical totals
  const int src = lane & (MAXWARPS - 1);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = (src < nwarps) ? buf[k * 32 + src] : 0.0;
#pragma unroll
  for (int off = MAXWARPS / 2; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  par ^= 1;
}

__device__ __forceinline__ double op_entry(double m, double k, double dt) {
  return __dadd_rn(m, __dmul_rn(dt, k));
}

__device__ __forceinline__ double grid_time(double t_base, int64_t g, double dt) {
  return __dadd_rn(t_base, __dmul_rn((double)g, dt));
}

__device__ __forceinline__ void write_status(int32_t* status, int slot, int code, int step,
                                             int interval, int iteration) {
  if (status == nullptr || slot < 0) return;
  int32_t* s = status + (int64_t)slot * kStatusInts;
  s[0] = code;
  s[1] = step;
  s[2] = interval;
  s[3] = iteration;
}

// ------------------------------------------------------------------ host
int small_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* M,
                    const double* K, const double* profile, double omega, double rtol,
                    int max_it, double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                    const int32_t* active, int64_t* elapsed, const double* xss,
                    cudaStream_t stream);

size_t fused_workspace_bytes(int S, int m, int k_max);
int small_run_fused(Ctx* ctx, int S, const double* M, const double* K, const double* profile,
                    double omega, double rtol, int max_it, const mlmcp_task_arrays& ar,
                    const mlmcp_parareal_batch& pr, int grid_ctas, void* ws, size_t ws_bytes,
                    cudaStream_t stream);

int small_periodic(Ctx* ctx, int n, const int32_t* sample, const double* dt, const double* M,
                   const double* K, const double* profile, double omega, double rtol,
                   int max_it, double* X, int32_t* iters, cudaStream_t stream);

int small_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                          const double* profile, double omega, double dt_c, double t0,
                          const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                          int max_it, double* U, const double* F, double* C, int32_t* iters,
                          int32_t* status, const int32_t* active, int64_t* elapsed,
                          const double* xss, cudaStream_t stream);

// direct path (dense LU per task, n <= MLMCP_DIRECT_MAX_ROWS)
int direct_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* M,
                     const double* K, const double* profile, double omega, double* xbuf,
                     double* qoi, int32_t* iters, int32_t* status, const int32_t* active,
                     int64_t* elapsed, cudaStream_t stream);

int direct_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                           const double* profile, double omega, double dt_c, double t0,
                           const int64_t* slice_k0, const int32_t* slice_steps, double* U,
                           const double* F, double* C, int32_t* status, const int32_t* active,
                           int64_t* elapsed, cudaStream_t stream);

int draw_uniform_device(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                        const double* lo, const double* range, double* out, cudaStream_t stream);
void draw_uniform_cpu(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                      const double* lo, const double* range, double* out);

size_t stream_workspace_bytes(const Ctx* ctx, int n_tasks, int S);
size_t stream_periodic_workspace_bytes(const Ctx* ctx, int n);
int stream_periodic(Ctx* ctx, int n, const int32_t* sample, const double* dt, const double* M,
                    const double* K, const double* rpar, const double* profile, double omega,
                    double rtol, int max_it, double* X, int32_t* iters, void* ws,
                    size_t ws_bytes, cudaStream_t stream);

int stream_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, int S, const double* M,
                     const double* K, const double* rpar, const double* profile, double omega, double rtol,
                     int max_it, const double* xss, double* xbuf, double* qoi, int32_t* iters,
                     int32_t* status, const int32_t* active, int64_t* elapsed, void* ws,
                     size_t ws_bytes, cudaStream_t stream);

int stream_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                           const double* rpar, const double* profile, double omega, double dt_c, double t0,
                           const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                           int max_it, double* U, const double* F, double* C, int32_t* iters,
                           int32_t* status, const int32_t* active, void* ws, size_t ws_bytes,
                           cudaStream_t stream);

// MLMCP_PATH_* of a streaming batch (stream_propagate's dispatch)
int stream_path_of(const Ctx* ctx, int n_tasks, int S, bool with_ss, bool with_rp,
                   bool correction);

size_t coop_workspace_bytes(const Ctx* ctx, int n_tasks);
bool coop_usable(const Ctx* ctx, int n_tasks);
// cluster path (one thread-block cluster per task, grids up to 128 x 128)
bool cluster_usable(const Ctx* ctx);
bool band_usable(const Ctx* ctx);
size_t band_ring_bytes(int n_tasks);
int band_max_signatures(const uint8_t* cls, int wd, int gh);
int band_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, const double* rpar,
                   const double* profile, double omega, double rtol, int max_it, int order,
                   int ls_on, const double* xss, double* ring, double* xbuf, double* qoi,
                   int32_t* iters, int32_t* status, const int32_t* active, int64_t* elapsed,
                   cudaStream_t stream);
int cluster_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks, int S, const double* M,
                      const double* K, const double* profile, double omega, double rtol,
                      int max_it, double* xbuf, double* qoi, int32_t* iters, int32_t* status,
                      const int32_t* active, int64_t* elapsed, void* ws, size_t ws_bytes,
                      cudaStream_t stream);
int cluster_parareal_coarse(Ctx* ctx, int S, int k, int m, const double* M, const double* K,
                            const double* profile, double omega, double dt_c, double t0,
                            const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                            int max_it, double* U, const double* F, double* C, int32_t* status,
                            const int32_t* active, cudaStream_t stream);
int coop_propagate(Ctx* ctx, int n_tasks, const mlmcp_task* tasks_d,
                   const std::vector<mlmcp_task>& h, int S, const double* A,
                   const double* dinv, const double* M, const double* K,
                   const double* profile, double omega, double rtol, int max_it, double* xbuf,
                   double* qoi, int32_t* iters, int32_t* status, const int32_t* active,
                   char* ws, size_t ws_bytes, cudaStream_t stream);

inline bool use_direct(const Ctx* ctx) {
  if (ctx->path == 3) return true;
  return ctx->path == 0 && ctx->n <= MLMCP_DIRECT_MAX_ROWS;
}

inline bool use_small(const Ctx* ctx) {
  if (ctx->path == 1) return true;
  if (ctx->path == 2 || ctx->path == 3) return false;
  return ctx->n <= kSmallMaxRows;
}

// device clock in ns (for the executor's effort accounting)
__device__ __forceinline__ int64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return (int64_t)t;
}

__device__ __forceinline__ void add_elapsed(int64_t* elapsed, int slot, int64_t t_start) {
  if (elapsed != nullptr && slot >= 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(elapsed + slot),
              (unsigned long long)(global_ns() - t_start));
}

}  // namespace mlmcp
