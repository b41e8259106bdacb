// Grid-barrier latency probe on all SMs (cooperative launch): counter barrier
// (one atomic per CTA on one word) vs flag barrier (CTA b writes flag[b]; CTA 0
// gathers with one warp and releases a generation word).
#include <cstdio>
#include <cuda_runtime.h>

__device__ void bar_counter(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) { atomicExch(bar, 0u); __threadfence(); atomicAdd(bar + 1, 1u); }
    else while (*gen == g) {}
    __threadfence();
  }
  __syncthreads();
}

__device__ void bar_flags(unsigned* flags, unsigned* rel, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) { __threadfence(); ((volatile unsigned*)flags)[blockIdx.x] = epoch; }
  if (blockIdx.x == 0) {
    for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
      while (((volatile unsigned*)flags)[b] != epoch) {}
    __syncthreads();
    if (threadIdx.x == 0) { __threadfence(); *(volatile unsigned*)rel = epoch; }
  } else if (threadIdx.x == 0) {
    while (*(volatile unsigned*)rel != epoch) {}
  }
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
}

__global__ void probe(unsigned* bar, unsigned* flags, unsigned* rel, long long* out, int n, int mode) {
  long long t0 = clock64();
  for (int i = 1; i <= n; ++i) {
    if (mode == 0) bar_counter(bar); else bar_flags(flags, rel, (unsigned)i);
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[mode] = t1 - t0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *bar, *flags, *rel; long long* out;
  cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  cudaMalloc(&flags, 4 * 1024); cudaMemset(flags, 0, 4096);
  cudaMalloc(&rel, 4); cudaMemset(rel, 0, 4);
  cudaMalloc(&out, 16);
  int n = 2000;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(flags, 0, 4096); cudaMemset(rel, 0, 4);
    void* args[] = {&bar, &flags, &rel, &out, &n, &mode};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, dim3(sms), dim3(256), args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %s: %s, %.2f us per barrier (%d CTAs)\n", mode ? "flags" : "counter",
           cudaGetErrorString(e), 1000.0 * ms / n, sms);
  }
  return 0;
}
