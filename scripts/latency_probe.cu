// Dependent-chain latency probe (cycles per op) for the ops on the PCG critical
// path: DFMA, DADD, 64-bit SHFL (2x32), LDS.64, MUFU.RCP64H, BAR (8 warps).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  sm[t] = t * 1.0;
  __syncthreads();
  double x = out[t], y = 1.0000001, z = 0.9999999;
  long long c0, c1;
  // DFMA chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = fma(x, y, z); x = fma(x, y, z); x = fma(x, y, z); x = fma(x, y, z); }
  c1 = clock64();
  if (t == 0) cyc[0] = (c1 - c0);
  // DADD chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = x + y; x = x + z; x = x + y; x = x + z; }
  c1 = clock64();
  if (t == 0) cyc[1] = (c1 - c0);
  // SHFL (double) + DADD chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4); x += __shfl_xor_sync(0xffffffffu, x, 8);
  }
  c1 = clock64();
  if (t == 0) cyc[2] = (c1 - c0);
  // LDS chain (pointer chasing through smem index)
  int idx = t;
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    idx = ((int)sm[idx] + 1) & 255; idx = ((int)sm[idx] + 1) & 255;
    idx = ((int)sm[idx] + 1) & 255; idx = ((int)sm[idx] + 1) & 255;
  }
  c1 = clock64();
  if (t == 0) cyc[3] = (c1 - c0);
  // rcp.approx chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0;
  }
  c1 = clock64();
  if (t == 0) cyc[4] = (c1 - c0);
  // barrier chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  c1 = clock64();
  if (t == 0) cyc[5] = (c1 - c0);
  out[t] = x + idx;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMemset(out, 0, 1024 * 8);
  cudaMalloc(&cyc, 64 * 8);
  const int n = 1000;
  const char* names[] = {"DFMA", "DADD", "SHFL64+DADD", "LDS+cvt+and", "RCP64+DADD", "BAR(256 thr)"};
  const double per[] = {4, 4, 4, 4, 2, 4};
  for (int threads : {32, 256}) {
    probe<<<1, threads>>>(out, cyc, n);
    cudaDeviceSynchronize();
    long long h[6];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%d:", threads);
    for (int k = 0; k < 6; ++k) printf("  %s %.1f", names[k], h[k] / (n * per[k]));
    printf("  (cycles per dependent op)\n");
  }
  return 0;
}
