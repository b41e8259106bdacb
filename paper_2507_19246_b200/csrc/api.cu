// api.cu — the extern "C" surface of libmlmcp.so (see include/mlmcp.h) plus
// the small batched kernels that are not PCG: assembly (K1), the KL
// conductivity field, the Parareal defect / finalize (K5), the magnetic
// energy QoI (K6) and the MLMC level reduction (K7).
#include <math.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "mlmcp_internal.cuh"

namespace mlmcp {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int cuda_fail(cudaError_t err, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(err));
  (void)cudaGetLastError();   // a non-sticky error must not surface in a later launch check
  return MLMCP_ECUDA;
}

namespace {

int einval(const std::string& msg) {
  set_error(msg);
  return MLMCP_EINVAL;
}

template <typename T>
int upload(T** dst, const T* src, size_t n) {
  *dst = nullptr;
  if (n == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(dst), n * sizeof(T)));
  MLMCP_CUDA_CHECK(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return MLMCP_OK;
}

// ---------------------------------------------------------------- K1 assembly
// One thread per (sample, CSR entry); contributions summed in ascending
// element order (the gather map is sorted on the host).
__global__ void assemble_kernel(int S, int nnz, const int32_t* __restrict__ cptr,
                                const int32_t* __restrict__ celem,
                                const double* __restrict__ cmw, const double* __restrict__ ckw,
                                const double* __restrict__ sigma, int64_t sstride,
                                const int32_t* __restrict__ sidx, const double* __restrict__ nu,
                                int64_t nstride, const int32_t* __restrict__ nidx, double* M,
                                double* K) {
  const int s = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const double* sg = sigma + s * sstride;
  const double* nv = nu + s * nstride;
  double m = 0.0, k = 0.0;
  for (int c = cptr[q]; c < cptr[q + 1]; ++c) {
    const int e = celem[c];
    const double se = sg[sidx ? sidx[e] : e];
    const double ne = nv[nidx ? nidx[e] : e];
    m = __dadd_rn(m, __dmul_rn(se, cmw[c]));
    k = __dadd_rn(k, __dmul_rn(ne, ckw[c]));
  }
  M[(int64_t)s * nnz + q] = m;
  K[(int64_t)s * nnz + q] = k;
}

// sigma[s][e] = exp(log_sigma0 + scale * sum_k xi[s][k] basis[k][e])
__global__ void kl_sigma_kernel(int S, int E, int modes, const double* __restrict__ xi,
                                const double* __restrict__ basis, double log_s0, double scale,
                                double* out) {
  extern __shared__ double xs[];
  const int s = blockIdx.y;
  for (int k = threadIdx.x; k < modes; k += blockDim.x) xs[k] = xi[(int64_t)s * modes + k];
  __syncthreads();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double acc = 0.0;
  for (int k = 0; k < modes; ++k) acc = fma(xs[k], basis[(int64_t)k * E + e], acc);
  out[(int64_t)s * E + e] = exp(log_s0 + scale * acc);
}

// ---------------------------------------------------------------- K6 energy
__global__ void energy_kernel(int n_items, int N, int64_t nnz, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ col, const int32_t* __restrict__ sample,
                              const int64_t* __restrict__ xoff, const double* __restrict__ xbuf,
                              const double* __restrict__ K, double* out) {
  __shared__ double red[2 * 4 * 32];
  const int it = blockIdx.x;
  const double* x = xbuf + xoff[it];
  const double* Ks = K + (int64_t)sample[it] * nnz;
  double acc = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double kx = 0.0;
    for (int q = rp[i]; q < rp[i + 1]; ++q) kx = fma(Ks[q], x[col[q]], kx);
    acc = fma(x[i], kx, acc);
  }
  int par = 0;
  double v[1] = {acc};
  block_allsum<1>(v, red, par);
  if (threadIdx.x == 0) out[it] = 0.5 * v[0];
}

// ---------------------------------------------------------------- K5 defect
// parareal.py:93-103 + :198-207 for iteration k of each active sample.
__global__ void defect_kernel(int S, int k, int m, int k_max, int N, const double* __restrict__ U,
                              const double* __restrict__ F, double tol, int32_t* active,
                              int32_t* k_used, double* defect) {
  __shared__ double red[2 * 4 * 32];
  const int s = blockIdx.x;
  if (active[s] == 0) return;
  const int64_t n64 = N;
  double d = 0.0;
  int par = 0;
  for (int n = k; n < m; ++n) {
    const double* u = U + ((int64_t)s * (m + 1) + n) * n64;
    const double* f = F + ((int64_t)s * (m + 1) + n) * n64;
    double jj = 0.0, ff = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double diff = f[i] - u[i];
      jj = fma(diff, diff, jj);
      ff = fma(f[i], f[i], ff);
    }
    double v[2] = {jj, ff};
    block_allsum<2>(v, red, par);
    const double ratio = sqrt(v[0]) / fmax(sqrt(v[1]), 1e-30);
    // np.max propagates NaN; fmax would drop it
    if (isnan(ratio) || isnan(d)) d = NAN;
    else d = fmax(d, ratio);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    defect[(int64_t)s * k_max + (k - 1)] = d;
    k_used[s] = k;
    if (d <= tol) active[s] = 0;
  }
}

__global__ void finalize_kernel(int S, int m, int N, double* U, const double* F,
                                const int32_t* k_used) {
  const int s = blockIdx.y;
  const int64_t n64 = N;
  const int ku = k_used[s];
  for (int n = ku; n <= m; ++n) {
    const int64_t o = ((int64_t)s * (m + 1) + n) * n64;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
      U[o + i] = F[o + i];
  }
}

// D[s][n] = U[s][n] (mode 0) or U[s][n] - D[s][n] (mode 1) for n = k-1 .. m-1
__global__ void delta_kernel(int S, int k, int m, int N, const double* U, double* D, int mode,
                             const int32_t* active) {
  const int s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int64_t n64 = N;
  for (int n = max(k - 1, 0); n < m; ++n) {
    const int64_t o = ((int64_t)s * (m + 1) + n) * n64;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
      D[o + i] = mode == 0 ? U[o + i] : U[o + i] - D[o + i];
  }
}

// ---------------------------------------------------------------- K7 level reduce
// Fixed-order reduction: thread j sums samples j, j+1024, ... in order, then a
// fixed tree.  Bitwise independent of how the sample slots were filled.
__global__ void level_reduce_kernel(int n, const double* __restrict__ ql,
                                    const double* __restrict__ qlm1, double* out) {
  __shared__ double red[2 * 4 * 32];
  double sy = 0.0, sy2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double y = ql[i] - (qlm1 ? qlm1[i] : 0.0);
    sy += y;
    sy2 = fma(y, y, sy2);
  }
  int par = 0;
  double v[2] = {sy, sy2};
  block_allsum<2>(v, red, par);
  if (threadIdx.x == 0) {
    const double mean = v[0] / n;
    out[0] = v[0];
    out[1] = v[1];
    out[2] = mean;
    out[3] = n > 1 ? (v[1] - n * mean * mean) / (n - 1) : 0.0;
  }
}

// sigma[s][r] = params[s][R + r] * mask[r]; rp[s][r] = (sigma[s][r], params[s][r])
__global__ void region_params_kernel(int S, int R, const double* __restrict__ params,
                                     const double* __restrict__ mask, double* sigma, double* rp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S * R) return;
  const int s = i / R, r = i % R;
  const double sg = __dmul_rn(params[(int64_t)s * 2 * R + R + r], mask ? mask[r] : 1.0);
  if (sigma) sigma[(int64_t)s * R + r] = sg;
  if (rp) {
    rp[((int64_t)s * R + r) * 2] = sg;
    rp[((int64_t)s * R + r) * 2 + 1] = params[(int64_t)s * 2 * R + r];
  }
}
}  // namespace
}  // namespace mlmcp

using namespace mlmcp;

struct mlmcp_ctx : public mlmcp::Ctx {};

extern "C" {

int mlmcp_abi_version(void) { return MLMCP_ABI_VERSION; }

const char* mlmcp_last_error(void) { return g_last_error.c_str(); }

uint64_t mlmcp_launch_count(void) { return g_launches.load(); }

int mlmcp_ctx_create(int device, int n_rows, int nnz, const int32_t* row_ptr,
                     const int32_t* col, mlmcp_ctx** out) {
  if (out == nullptr) return einval("out is null");
  *out = nullptr;
  if (n_rows < 1 || nnz < 1 || row_ptr == nullptr || col == nullptr)
    return einval("empty or null sparsity pattern");
  if (row_ptr[0] != 0 || row_ptr[n_rows] != nnz) return einval("row_ptr must span [0, nnz]");
  int max_row = 0;
  for (int i = 0; i < n_rows; ++i) {
    const int len = row_ptr[i + 1] - row_ptr[i];
    if (len < 1) return einval("row " + std::to_string(i) + " is empty (no diagonal)");
    if (len > kMaxNz)
      return einval("row " + std::to_string(i) + " has " + std::to_string(len) +
                    " entries; the kernels accept at most 8");
    bool diag = false;
    for (int q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      if (col[q] < 0 || col[q] >= n_rows) return einval("column index out of range");
      if (q > row_ptr[i] && col[q] <= col[q - 1]) return einval("columns must be sorted and unique");
      diag |= col[q] == i;
    }
    if (!diag) return einval("row " + std::to_string(i) + " has no diagonal entry");
    max_row = std::max(max_row, len);
  }
  int ndev = 0;
  MLMCP_CUDA_CHECK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return einval("invalid device ordinal");
  MLMCP_CUDA_CHECK(cudaSetDevice(device));
  auto* c = new mlmcp_ctx();
  c->device = device;
  c->n = n_rows;
  c->nnz = nnz;
  c->max_row_nnz = max_row;
  std::vector<int32_t> ell_col((size_t)max_row * n_rows), ell_pos((size_t)max_row * n_rows);
  for (int i = 0; i < n_rows; ++i) {
    const int len = row_ptr[i + 1] - row_ptr[i];
    for (int j = 0; j < max_row; ++j) {
      const bool in = j < len;
      ell_col[(size_t)j * n_rows + i] = in ? col[row_ptr[i] + j] : i;
      ell_pos[(size_t)j * n_rows + i] = in ? row_ptr[i] + j : -1;
    }
  }
  // uniform-offset stencil detection
  {
    std::vector<int> offs;
    bool stencil = true;
    for (int i = 0; i < n_rows && stencil; ++i)
      for (int q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
        const int d = col[q] - i;
        if (std::find(offs.begin(), offs.end(), d) == offs.end()) {
          offs.push_back(d);
          if ((int)offs.size() > kMaxNz) { stencil = false; break; }
        }
      }
    if (stencil) {
      std::sort(offs.begin(), offs.end());
      c->stencil_w = (int)offs.size();
      int pad = 0;
      for (int k = 0; k < c->stencil_w; ++k) {
        c->stencil_off[k] = offs[k];
        pad = std::max(pad, std::abs(offs[k]));
      }
      c->stencil_pad = pad;
    }
  }
  std::vector<int32_t> spos((size_t)std::max(c->stencil_w, 1) * n_rows, -1);
  for (int i = 0; i < n_rows && c->stencil_w; ++i)
    for (int q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
      const int d = col[q] - i;
      const int k = (int)(std::find(c->stencil_off, c->stencil_off + c->stencil_w, d) - c->stencil_off);
      spos[(size_t)k * n_rows + i] = q;
    }
  // 2D grid detection (structured FE mesh small enough for the grid-tiled kernel)
  std::vector<int32_t> gpos;
  for (int wd = 2; wd <= 32 && c->grid_wd == 0; ++wd) {
    if (n_rows % wd != 0 || n_rows / wd > 32) continue;
    std::vector<int32_t> g((size_t)7 * n_rows, -1);
    bool ok = true;
    for (int i = 0; i < n_rows && ok; ++i) {
      const int x = i % wd, y = i / wd;
      for (int q = row_ptr[i]; q < row_ptr[i + 1] && ok; ++q) {
        const int j = col[q], xj = j % wd, yj = j / wd;
        const int dx = xj - x, dy = yj - y;
        int slot = -1;
        if (dx == -1 && dy == -1) slot = 0;
        else if (dx == 0 && dy == -1) slot = 1;
        else if (dx == -1 && dy == 0) slot = 2;
        else if (dx == 0 && dy == 0) slot = 3;
        else if (dx == 1 && dy == 0) slot = 4;
        else if (dx == 0 && dy == 1) slot = 5;
        else if (dx == 1 && dy == 1) slot = 6;
        if (slot < 0) ok = false;
        else g[(size_t)slot * n_rows + i] = q;
      }
    }
    if (ok) {
      c->grid_wd = wd;
      c->grid_h = n_rows / wd;
      gpos.swap(g);
    }
  }
  // the same detection for larger grids (the cluster path up to 128 x 128, the
  // tile path of the streaming kernels beyond), when the pattern is too large
  // for the single-SM kernel
  std::vector<int32_t> cpos;
  for (int wd = 2; wd <= 4096 && c->cl_wd == 0 && n_rows > kSmallMaxRows; ++wd) {
    if (n_rows % wd != 0 || n_rows / wd > 4096) continue;
    std::vector<int32_t> g((size_t)7 * n_rows, -1);
    bool ok = true;
    for (int i = 0; i < n_rows && ok; ++i) {
      const int x = i % wd, y = i / wd;
      for (int q = row_ptr[i]; q < row_ptr[i + 1] && ok; ++q) {
        const int j = col[q], dx = j % wd - x, dy = j / wd - y;
        int slot = -1;
        if (dx == -1 && dy == -1) slot = 0;
        else if (dx == 0 && dy == -1) slot = 1;
        else if (dx == -1 && dy == 0) slot = 2;
        else if (dx == 0 && dy == 0) slot = 3;
        else if (dx == 1 && dy == 0) slot = 4;
        else if (dx == 0 && dy == 1) slot = 5;
        else if (dx == 1 && dy == 1) slot = 6;
        if (slot < 0) ok = false;
        else g[(size_t)slot * n_rows + i] = q;
      }
    }
    if (ok) {
      c->cl_wd = wd;
      c->cl_h = n_rows / wd;
      cpos.swap(g);
    }
  }
  int rc = upload(&c->row_ptr, row_ptr, (size_t)n_rows + 1);
  if (!rc && c->cl_wd) rc = upload(&c->cl_pos, cpos.data(), cpos.size());
  if (!rc && c->stencil_w) rc = upload(&c->stencil_pos, spos.data(), spos.size());
  if (!rc && c->grid_wd) rc = upload(&c->grid_pos, gpos.data(), gpos.size());
  if (!rc) rc = upload(&c->col, col, (size_t)nnz);
  if (!rc) rc = upload(&c->ell_col, ell_col.data(), ell_col.size());
  if (!rc) rc = upload(&c->ell_pos, ell_pos.data(), ell_pos.size());
  if (!rc) {
    cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&c->host_counters), 64);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocHost");
  }
  if (!rc) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&c->grid_bar), (1 + 1024) * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(c->grid_bar, 0, (1 + 1024) * sizeof(unsigned int));
    if (e != cudaSuccess) rc = cuda_fail(e, "grid barrier allocation");
  }
  if (rc) {
    mlmcp_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return MLMCP_OK;
}

int mlmcp_ctx_destroy(mlmcp_ctx* c) {
  if (c == nullptr) return MLMCP_OK;
  cudaSetDevice(c->device);
  cudaFree(c->row_ptr);
  cudaFree(c->col);
  cudaFree(c->ell_col);
  cudaFree(c->ell_pos);
  cudaFree(c->stencil_pos);
  cudaFree(c->grid_pos);
  cudaFree(c->cl_pos);
  cudaFree(c->grid_bar);
  cudaFree(c->cptr);
  cudaFree(c->celem);
  cudaFree(c->cmw);
  cudaFree(c->ckw);
  cudaFree(c->rcls);
  cudaFree(c->rckey);
  if (c->host_counters) cudaFreeHost(c->host_counters);
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  for (cudaEvent_t e : c->iter_ev)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : c->cap_stream)
    if (s) cudaStreamDestroy(s);
  delete c;
  return MLMCP_OK;
}

int mlmcp_ctx_info(const mlmcp_ctx* c, int* max_row_nnz, int* small_max_rows) {
  if (c == nullptr) return einval("null context");
  if (max_row_nnz) *max_row_nnz = c->max_row_nnz;
  if (small_max_rows) *small_max_rows = kSmallMaxRows;
  return MLMCP_OK;
}

int mlmcp_ctx_set_path(mlmcp_ctx* c, int path) {
  if (c == nullptr) return einval("null context");
  if (path < 0 || path > 3)
    return einval("path must be 0 (auto), 1 (SM-resident), 2 (streaming) or 3 (direct)");
  if (path == 1 && c->n > kSmallMaxRows)
    return einval("SM-resident path holds at most 1024 rows");
  if (path == 3 && c->n > MLMCP_DIRECT_MAX_ROWS)
    return einval("direct path holds at most MLMCP_DIRECT_MAX_ROWS rows");
  c->path = path;
  return MLMCP_OK;
}

int mlmcp_stream_timing(mlmcp_ctx* c, int mode, double* ms, int64_t* launches) {
  if (c == nullptr) return einval("null context");
  if (mode != 0 && mode != 1) return einval("mode must be 0 (stop) or 1 (reset and start)");
  if (mode == 1) {
    MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
    for (auto& e : c->iter_ev)
      if (e == nullptr) MLMCP_CUDA_CHECK(cudaEventCreate(&e));
    c->iter_ms = 0.0;
    c->iter_launches = 0;
  }
  c->time_iters = mode;
  if (ms) *ms = c->iter_ms;
  if (launches) *launches = c->iter_launches;
  return MLMCP_OK;
}

int mlmcp_ctx_set_assembly(mlmcp_ctx* c, int n_elem, int n_contrib, const int32_t* cptr,
                           const int32_t* elem, const double* mw, const double* kw) {
  if (c == nullptr) return einval("null context");
  if (n_elem < 1 || n_contrib < 1 || !cptr || !elem || !mw || !kw)
    return einval("empty assembly map");
  if (cptr[0] != 0 || cptr[c->nnz] != n_contrib) return einval("cptr must span [0, n_contrib]");
  for (int q = 0; q < c->nnz; ++q)
    if (cptr[q + 1] < cptr[q]) return einval("cptr must be non-decreasing");
  for (int i = 0; i < n_contrib; ++i)
    if (elem[i] < 0 || elem[i] >= n_elem) return einval("element index out of range");
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  cudaFree(c->cptr);
  cudaFree(c->celem);
  cudaFree(c->cmw);
  cudaFree(c->ckw);
  c->n_elem = n_elem;
  c->n_contrib = n_contrib;
  int rc = upload(&c->cptr, cptr, (size_t)c->nnz + 1);
  if (!rc) rc = upload(&c->celem, elem, (size_t)n_contrib);
  if (!rc) rc = upload(&c->cmw, mw, (size_t)n_contrib);
  if (!rc) rc = upload(&c->ckw, kw, (size_t)n_contrib);
  return rc;
}

int mlmcp_ctx_set_region_grid(mlmcp_ctx* c, int n_regions, const uint32_t* code,
                              const double* mw, const double* kw) {
  if (c == nullptr) return einval("null context");
  if (n_regions == 0) {   // unregister
    cudaSetDevice(c->device);
    cudaFree(c->rcls);
    cudaFree(c->rckey);
    c->rcls = nullptr;
    c->rckey = nullptr;
    c->rC = 0;
    c->rR = 0;
    c->band_sigs = 0;
    return MLMCP_OK;
  }
  if (n_regions < 1 || n_regions > 16 || !code || !mw || !kw)
    return einval("region grid: need 1..16 regions and code / weight arrays");
  if (c->cl_wd == 0 || (int64_t)c->cl_wd * c->cl_h != c->n)
    return einval("region grid: the pattern is not a structured 2D grid");
  for (int i = 0; i < c->n; ++i)
    for (int e = 0; e < 6; ++e)
      if ((int)((code[i] >> (4 * e)) & 15u) >= n_regions)
        return einval("region grid: triangle region index out of range");
  // classes: distinct (code, neighbour mask) keys; the mask bits say which of
  // the SW, S, W, E, N, NE neighbours are interior points (Dirichlet rows drop
  // the others).  More than 256 classes: no region mode (stored operator).
  std::vector<uint8_t> cls((size_t)c->n);
  std::vector<uint32_t> keys;
  {
    std::unordered_map<uint32_t, int> idx;
    const int wd = c->cl_wd, gh = c->cl_h;
    for (int i = 0; i < c->n && keys.size() <= 256; ++i) {
      const int gx = i % wd, gy = i / wd;
      const bool w = gx > 0, s = gy > 0, e = gx + 1 < wd, n = gy + 1 < gh;
      const uint32_t mask = (uint32_t)(w && s) | ((uint32_t)s << 1) | ((uint32_t)w << 2) |
                            ((uint32_t)e << 3) | ((uint32_t)n << 4) | ((uint32_t)(e && n) << 5);
      const uint32_t key = (code[i] & 0x00ffffffu) | (mask << 24);
      auto it = idx.find(key);
      if (it == idx.end()) {
        it = idx.emplace(key, (int)keys.size()).first;
        keys.push_back(key);
      }
      cls[(size_t)i] = (uint8_t)(it->second & 255);
    }
  }
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  cudaFree(c->rcls);
  cudaFree(c->rckey);
  c->rcls = nullptr;
  c->rckey = nullptr;
  c->rC = 0;
  c->band_sigs = 0;
  if (keys.size() <= 256) {
    MLMCP_CUDA_CHECK(cudaMalloc(&c->rcls, (size_t)c->n));
    MLMCP_CUDA_CHECK(cudaMemcpy(c->rcls, cls.data(), (size_t)c->n, cudaMemcpyHostToDevice));
    MLMCP_CUDA_CHECK(cudaMalloc(&c->rckey, sizeof(uint32_t) * keys.size()));
    MLMCP_CUDA_CHECK(cudaMemcpy(c->rckey, keys.data(), sizeof(uint32_t) * keys.size(),
                                cudaMemcpyHostToDevice));
    c->rC = (int)keys.size();
    c->band_sigs = band_max_signatures(cls.data(), c->cl_wd, c->cl_h);
  }
  for (int i = 0; i < 12; ++i) {
    c->rmw[i] = mw[i];
    c->rkw[i] = kw[i];
  }
  c->rR = n_regions;
  return MLMCP_OK;
}


int mlmcp_region_params(int S, int R, const double* params, const double* mask, double* sigma,
                        double* rp, void* stream) {
  if (S < 0 || R < 1 || R > 16 || !params || (!sigma && !rp)) return einval("bad region parameters");
  if (S == 0) return MLMCP_OK;
  region_params_kernel<<<(S * R + 255) / 256, 256, 0, (cudaStream_t)stream>>>(S, R, params, mask,
                                                                            sigma, rp);
  MLMCP_LAUNCH_CHECK("region_params_kernel");
  return MLMCP_OK;
}

int mlmcp_assemble(mlmcp_ctx* c, int S, const double* sigma, int64_t sstride,
                   const int32_t* sidx, const double* nu, int64_t nstride, const int32_t* nidx,
                   double* M, double* K, void* stream) {
  if (c == nullptr) return einval("null context");
  if (c->cptr == nullptr) return einval("assembly map not set (mlmcp_ctx_set_assembly)");
  if (S < 0 || !sigma || !nu || !M || !K) return einval("null assembly argument");
  if (S == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  dim3 grid((c->nnz + 255) / 256, S);
  assemble_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      S, c->nnz, c->cptr, c->celem, c->cmw, c->ckw, sigma, sstride, sidx, nu, nstride, nidx, M, K);
  MLMCP_LAUNCH_CHECK("assemble_kernel");
  return MLMCP_OK;
}

int mlmcp_kl_sigma(int S, int E, int modes, const double* xi, const double* basis,
                   double log_s0, double scale, double* out, void* stream) {
  if (S < 0 || E < 1 || modes < 1 || modes > 4096 || !xi || !basis || !out)
    return einval("bad KL arguments");
  if (S == 0) return MLMCP_OK;
  dim3 grid((E + 255) / 256, S);
  kl_sigma_kernel<<<grid, 256, modes * sizeof(double), (cudaStream_t)stream>>>(
      S, E, modes, xi, basis, log_s0, scale, out);
  MLMCP_LAUNCH_CHECK("kl_sigma_kernel");
  return MLMCP_OK;
}

size_t mlmcp_workspace_bytes(const mlmcp_ctx* c, int n_tasks, int S) {
  if (c == nullptr || use_small(c) || use_direct(c)) return 0;
  const size_t base = stream_workspace_bytes(c, std::max(n_tasks, S), S);
  // coarse sweep extras: tasks + cval + tstatus
  const size_t extra = ((sizeof(mlmcp_task) * S + 255) & ~size_t(255)) +
                       ((sizeof(double) * (size_t)S * c->n + 255) & ~size_t(255)) +
                       ((sizeof(int32_t) * 4 * S + 255) & ~size_t(255));
  return base + extra;
}

int mlmcp_propagate(mlmcp_ctx* c, int n_tasks, const mlmcp_task* tasks, int S, const double* M,
                    const double* K, const double* rpar, const double* profile, double omega,
                    double rtol,
                    int max_it, const double* xss, double* xbuf, double* qoi, int32_t* iters,
                    int32_t* status, const int32_t* active, int64_t* elapsed, void* ws,
                    size_t ws_bytes, void* stream) {
  if (c == nullptr) return einval("null context");
  if (n_tasks < 0 || S < 1 || !tasks || !M || !K || !profile || !xbuf)
    return einval("null or empty propagate argument");
  if (!(rtol > 0.0) || max_it < 1) return einval("rtol must be > 0 and max_it >= 1");
  if (n_tasks == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  if (use_direct(c))
    return direct_propagate(c, n_tasks, tasks, M, K, profile, omega, xbuf, qoi, iters, status,
                            active, elapsed, (cudaStream_t)stream);
  if (use_small(c))
    return small_propagate(c, n_tasks, tasks, M, K, profile, omega, rtol, max_it, xbuf, qoi,
                           iters, status, active, elapsed, xss, (cudaStream_t)stream);
  return stream_propagate(c, n_tasks, tasks, S, M, K, rpar, profile, omega, rtol, max_it, xss, xbuf,
                          qoi, iters, status, active, elapsed, ws, ws_bytes,
                          (cudaStream_t)stream);
}

int mlmcp_parareal_coarse(mlmcp_ctx* c, int S, int k, int m, const double* M, const double* K,
                          const double* rpar, const double* profile, double omega, double dt_c,
                          double t0,
                          const int64_t* slice_k0, const int32_t* slice_steps, double rtol,
                          int max_it, double* U, const double* F, double* C, int32_t* iters,
                          int32_t* status, const int32_t* active, int64_t* elapsed,
                          const double* xss, void* ws, size_t ws_bytes, void* stream) {
  if (c == nullptr) return einval("null context");
  if (S < 0 || m < 1 || k < 1 || k > m || !M || !K || !profile || !slice_k0 || !slice_steps ||
      !U || !F || !C || !active || !status)
    return einval("bad Parareal coarse arguments");
  if (!(rtol > 0.0) || max_it < 1 || !(dt_c > 0.0)) return einval("bad solver tolerances");
  if (S == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  if (use_direct(c))
    return direct_parareal_coarse(c, S, k, m, M, K, profile, omega, dt_c, t0, slice_k0,
                                  slice_steps, U, F, C, status, active, elapsed,
                                  (cudaStream_t)stream);
  if (use_small(c))
    return small_parareal_coarse(c, S, k, m, M, K, profile, omega, dt_c, t0, slice_k0,
                                 slice_steps, rtol, max_it, U, F, C, iters, status, active,
                                 elapsed, xss, (cudaStream_t)stream);
  return stream_parareal_coarse(c, S, k, m, M, K, rpar, profile, omega, dt_c, t0, slice_k0,
                                slice_steps, rtol, max_it, U, F, C, iters, status, active, ws,
                                ws_bytes, (cudaStream_t)stream);
}

size_t mlmcp_periodic_workspace_bytes(const mlmcp_ctx* c, int n) {
  if (c == nullptr || n <= 0 || use_small(c) || use_direct(c)) return 0;
  return stream_periodic_workspace_bytes(c, n);
}

int mlmcp_periodic_state(mlmcp_ctx* c, int n, const int32_t* sample, const double* dt, int S,
                         const double* M, const double* K, const double* rpar,
                         const double* profile, double omega,
                         double rtol, int max_it, double* X, int32_t* iters, void* ws,
                         size_t ws_bytes, void* stream) {
  if (c == nullptr) return einval("null context");
  if (n < 0 || S < 1 || !sample || !dt || !M || !K || !profile || !X)
    return einval("null or empty periodic-state argument");
  if (!(rtol > 0.0) || max_it < 1) return einval("rtol must be > 0 and max_it >= 1");
  if (use_direct(c)) return einval("periodic steady states: not on the direct path");
  if (n == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  if (use_small(c))
    return small_periodic(c, n, sample, dt, M, K, profile, omega, rtol, max_it, X, iters,
                          (cudaStream_t)stream);
  return stream_periodic(c, n, sample, dt, M, K, rpar, profile, omega, rtol, max_it, X, iters,
                         ws, ws_bytes, (cudaStream_t)stream);
}

size_t mlmcp_fused_workspace_bytes(int S, int m, int k_max) {
  if (S < 0 || m < 0 || k_max < 0) return 0;
  return fused_workspace_bytes(S, std::max(m, 1), std::max(k_max, 1));
}

int mlmcp_run_fused(mlmcp_ctx* c, int S, const double* M, const double* K, const double* profile,
                    double omega, double rtol, int max_it, const mlmcp_task_arrays* ar,
                    const mlmcp_parareal_batch* pr, int grid_ctas, void* ws, size_t ws_bytes,
                    void* stream) {
  if (c == nullptr || ar == nullptr || pr == nullptr) return einval("null fused argument");
  if (grid_ctas < 0) return einval("grid_ctas must be >= 0");
  if (S < 1 || !M || !K || !profile) return einval("null or empty operator arrays");
  if (!(rtol > 0.0) || max_it < 1) return einval("rtol must be > 0 and max_it >= 1");
  if (use_direct(c) || !use_small(c)) return einval("the fused launch needs the SM-resident path");
  if (ar->n_seq < 0 || !ar->xbuf_d || (ar->n_seq > 0 && !ar->seq_tasks_d))
    return einval("bad task arrays");
  if (pr->S < 0 || (pr->S > 0 && (pr->m < 1 || pr->k_max < 1 || pr->k_max > pr->m ||
                                  pr->row0 < 0 || pr->row0 + pr->S > S || !pr->fine_tasks_d ||
                                  !pr->C_d || !pr->slice_k0_d || !pr->slice_steps_d ||
                                  !ar->active_d || !ar->status_d || !pr->k_used_d ||
                                  !pr->defects_d || pr->u_off < 0 || pr->c_tmp_off < 0 ||
                                  pr->coarse_slot < 0 || !(pr->dt_c > 0.0))))
    return einval("bad Parareal batch");
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  return small_run_fused(c, S, M, K, profile, omega, rtol, max_it, *ar, *pr, grid_ctas, ws,
                         ws_bytes, (cudaStream_t)stream);
}

int mlmcp_draw_uniform(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                       const double* lo, const double* range, double* out, void* stream) {
  if (n < 0 || P < 1 || k_first < 0 || (n > 0 && (!lo || !range || !out)))
    return einval("bad draw arguments");
  return draw_uniform_device(seed, level, k_first, n, P, lo, range, out, (cudaStream_t)stream);
}

int mlmcp_draw_uniform_host(uint64_t seed, uint64_t level, int64_t k_first, int n, int P,
                            const double* lo, const double* range, double* out) {
  if (n < 0 || P < 1 || k_first < 0 || (n > 0 && (!lo || !range || !out)))
    return einval("bad draw arguments");
  draw_uniform_cpu(seed, level, k_first, n, P, lo, range, out);
  return MLMCP_OK;
}

int mlmcp_parareal_defect(mlmcp_ctx* c, int S, int k, int m, int k_max, const double* U,
                          const double* F, double tol, int32_t* active, int32_t* k_used,
                          double* defect, void* stream) {
  if (c == nullptr) return einval("null context");
  if (S < 0 || k < 1 || k > m || k_max < k || !U || !F || !active || !k_used || !defect)
    return einval("bad Parareal defect arguments");
  if (S == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  defect_kernel<<<S, 512, 0, (cudaStream_t)stream>>>(S, k, m, k_max, c->n, U, F, tol, active,
                                                      k_used, defect);
  MLMCP_LAUNCH_CHECK("defect_kernel");
  return MLMCP_OK;
}

int mlmcp_parareal_finalize(mlmcp_ctx* c, int S, int m, double* U, const double* F,
                            const int32_t* k_used, void* stream) {
  if (c == nullptr) return einval("null context");
  if (S < 0 || m < 1 || !U || !F || !k_used) return einval("bad finalize arguments");
  if (S == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  dim3 grid(std::min((c->n + 255) / 256, 64), S);
  finalize_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(S, m, c->n, U, F, k_used);
  MLMCP_LAUNCH_CHECK("finalize_kernel");
  return MLMCP_OK;
}

int mlmcp_parareal_delta(mlmcp_ctx* c, int S, int k, int m, const double* U, double* D, int mode,
                         const int32_t* active, void* stream) {
  if (c == nullptr) return einval("null context");
  if (S < 0 || m < 1 || k < 1 || k > m || !U || !D || (mode != 0 && mode != 1))
    return einval("bad Parareal delta arguments");
  if (S == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  dim3 grid(std::min((c->n + 255) / 256, 64), S);
  delta_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(S, k, m, c->n, U, D, mode, active);
  MLMCP_LAUNCH_CHECK("delta_kernel");
  return MLMCP_OK;
}

int mlmcp_propagate_path(const mlmcp_ctx* c, int n_tasks, int S, int with_ss, int with_rp,
                         int correction) {
  if (c == nullptr) return einval("null context");
  if (use_direct(c)) return MLMCP_PATH_DIRECT;
  if (use_small(c)) return MLMCP_PATH_SMALL;
  return stream_path_of(c, n_tasks, S, with_ss != 0, with_rp != 0, correction != 0);
}

int mlmcp_energy(mlmcp_ctx* c, int n, const int32_t* sample, const int64_t* xoff,
                 const double* xbuf, const double* K, double* out, void* stream) {
  if (c == nullptr) return einval("null context");
  if (n < 0 || !sample || !xoff || !xbuf || !K || !out) return einval("bad energy arguments");
  if (n == 0) return MLMCP_OK;
  MLMCP_CUDA_CHECK(cudaSetDevice(c->device));
  energy_kernel<<<n, 512, 0, (cudaStream_t)stream>>>(n, c->n, c->nnz, c->row_ptr, c->col, sample,
                                                      xoff, xbuf, K, out);
  MLMCP_LAUNCH_CHECK("energy_kernel");
  return MLMCP_OK;
}

int mlmcp_level_reduce(int n, const double* ql, const double* qlm1, double* out, void* stream) {
  if (n < 1 || !ql || !out) return einval("bad level-reduce arguments");
  level_reduce_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(n, ql, qlm1, out);
  MLMCP_LAUNCH_CHECK("level_reduce_kernel");
  return MLMCP_OK;
}

}  // extern "C"
